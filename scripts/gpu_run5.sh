cd $GRAFT_REPO_ROOT
python scripts/diag.py --config 3 > gpurun_out/d1_c3.log 2>&1
python scripts/diag.py --config 5 --iters 5 > gpurun_out/d1_c5.log 2>&1
python scripts/diag.py --config 4 > gpurun_out/d1_c4.log 2>&1
