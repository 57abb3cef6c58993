cd $GRAFT_REPO_ROOT
T=${1:-lean}
timeout 1200 python -m pytest tests/test_gpu_fast.py tests/test_gpu_fullsize.py tests/test_multi.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/${T}_bench_c3.log 2> gpurun_out/${T}_bench_c3.err
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_c5.log 2>&1
SSLIC_NO_LEAN=1 timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_c5_generic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assign_lean -s 9 -c 1 -o gpurun_out/${T}_lean_c3 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_c3.log 2>&1
