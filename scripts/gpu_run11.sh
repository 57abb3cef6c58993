cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -x -q > gpurun_out/r11_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r11_pytest.log
python scripts/diag.py --config 3 > gpurun_out/d7_c3.log 2>&1
python scripts/diag.py --config 4 > gpurun_out/d7_c4.log 2>&1
python scripts/diag.py --config 5 --iters 3 > gpurun_out/d7_c5.log 2>&1
python bench.py --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/p7_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 9 -c 1 -o gpurun_out/p7_assign python bench.py --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/p7_ncu.log 2>&1
