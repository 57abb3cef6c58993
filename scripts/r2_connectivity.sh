cd $GRAFT_REPO_ROOT
T=${1:-conn2}
timeout 1200 python -m pytest tests/test_gpu_connectivity.py tests/test_gpu_parity.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
export SSLIC_TIMING=1
timeout 900 python scripts/conn_time.py --config 3 --reps 2 --no-ref > gpurun_out/${T}_c3.log 2>&1
timeout 900 python scripts/conn_time.py --config 1 --reps 5 > gpurun_out/${T}_c1.log 2>&1
timeout 1800 python scripts/config5_segment.py > gpurun_out/${T}_c5full.log 2>&1; echo "exit $?" >> gpurun_out/${T}_c5full.log
