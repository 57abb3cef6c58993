cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/r2_smoke.log
timeout 600 python bench.py --steps 7 --warmup 3 --no-cpu > gpurun_out/r2_bench_c3.log 2>&1
timeout 600 python bench.py --config 4 --steps 7 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_c4.log 2>&1
timeout 600 python bench.py --config 2 --steps 7 --warmup 3 --no-cpu > gpurun_out/r2_bench_c2.log 2>&1
echo done
