cd $GRAFT_REPO_ROOT
python bench.py --config 2 --no-cpu > gpurun_out/g_b2a.log 2>&1
python bench.py --config 1 --no-cpu > gpurun_out/g_b2b.log 2>&1
python - > gpurun_out/g_e2e.log 2>&1 <<'PY'
import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1806_08741_b200 as s
dims=(2048,1216); ch=3
buf=torch.empty(dims[0]*dims[1]*ch, dtype=torch.float32, device='cuda')
s.synth_generate(2, dims, np.float32, ch, 5, 0, 1, buf.data_ptr()); torch.cuda.synchronize()
host=buf.cpu().numpy()
img=s.NDImage(dims, ch, host)
p=s.SlicParams(grid=[32,32], weight_m=10.0, max_iterations=10, enforce_connectivity=False)
for i in range(4):
    t=time.perf_counter(); r=s.run_slic(img,p); print('run_slic', time.perf_counter()-t)
PY
