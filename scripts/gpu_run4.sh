cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r4_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r4_pytest.log
timeout 600 python bench.py --steps 7 --warmup 3 --no-cpu --no-e2e > gpurun_out/r4_bench_c3.log 2>&1
timeout 600 python bench.py --config 4 --steps 7 --warmup 3 --no-cpu --no-e2e > gpurun_out/r4_bench_c4.log 2>&1
timeout 900 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r4_bench_c5.log 2>&1
echo done
