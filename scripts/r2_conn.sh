# connectivity timings (ours vs the reference on the same label maps)
cd $GRAFT_REPO_ROOT
T=${1:-conn}
export SSLIC_TIMING=1
timeout 600 python scripts/conn_time.py --config 1 --reps 5 > gpurun_out/${T}_c1.log 2>&1
timeout 900 python scripts/conn_time.py --config 5 --planes 3456 3520 --reps 2 > gpurun_out/${T}_c5sub.log 2>&1
timeout 1200 python scripts/conn_time.py --config 3 --reps 2 > gpurun_out/${T}_c3.log 2>&1
timeout 900 python scripts/conn_time.py --config 5 --planes 3328 3840 --reps 1 --no-ref > gpurun_out/${T}_c5_512.log 2>&1
