cd $GRAFT_REPO_ROOT
python scripts/conn_time.py --config 1 > gpurun_out/conn_c1.log 2>&1
python scripts/conn_time.py --config 2 > gpurun_out/conn_c2.log 2>&1
timeout 900 python scripts/conn_time.py --config 3 --ref-planes 64 > gpurun_out/conn_c3.log 2>&1
