# correctness subset + benches of configs 3, 4, 5 (device-only)
cd $GRAFT_REPO_ROOT
T=${1:-chk}
timeout 1500 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
for c in 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/${T}_bench_c$c.log 2>&1
done
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_c5.log 2>&1
python - "$T" <<'PY'
import json, sys, glob
t = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/{t}_bench_c[345].log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); r = d["roofline"]
            print(f, round(d["value"] / 1e9, 2), "Gvox/s frac", round(r["frac"], 4),
                  "evals", [round(x, 2) for x in r["algorithmic"]["evals_performed_per_voxel"]],
                  "ms/it", [round(x, 2) for x in r["kernel_ms_per_iteration"]])
PY
