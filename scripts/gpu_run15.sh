cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -x -q > gpurun_out/r22_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r22_pytest.log
python scripts/diag.py --config 3 > gpurun_out/d18_c3.log 2>&1
python scripts/diag.py --config 4 > gpurun_out/d18_c4.log 2>&1
python scripts/diag.py --config 5 --iters 4 > gpurun_out/d18_c5.log 2>&1
