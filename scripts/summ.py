import json, sys
for f in sys.argv[1:]:
    try:
        lines = [l for l in open(f).read().strip().splitlines() if l.startswith('{')]
        d = json.loads(lines[-1])
    except Exception as e:
        print(f, 'ERR', open(f).read()[-800:]); continue
    r = d.get('roofline') or {}
    al = r.get('algorithmic', {})
    print(f, round(d['value']/1e9, 2), 'Gvox/s', 'ms/step', round(d['ms_per_step'], 3),
          'kernel_ms', round(r.get('kernel_ms', 0), 3), 'frac', round(r.get('frac', 0), 3),
          'E', round(al.get('E_window_evals_per_voxel', 0), 2), 'evals', round(al.get('evals_performed_per_voxel', 0), 2),
          'redec', al.get('fp64_redecided_voxel_frac'), 'chg', al.get('label_changed_voxel_frac_last_iter'),
          'e2e', (d.get('e2e') or {}).get('value'), 'clk', d.get('clocks', {}).get('sm_mhz'))
