cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/r1_smi.txt 2>&1
nproc >> gpurun_out/r1_smi.txt; free -g >> gpurun_out/r1_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/r1_smoke.log
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/r1_bench_c1.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r1_bench_c3.log 2>&1
echo done
