cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/conn2_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/conn2_pytest.log
python scripts/conn_time.py --config 1 > gpurun_out/conn2_c1.log 2>&1
timeout 900 python scripts/conn_time.py --config 3 > gpurun_out/conn2_c3.log 2>&1
