cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/b6_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/b6_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b6_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/b6_smoke.log
python bench.py > gpurun_out/b6_bench_c3.log 2>&1
python bench.py --impl reference > gpurun_out/b6_ref_c3.log 2>&1
python bench.py --config 5 --steps 2 --warmup 3 --no-e2e > gpurun_out/b6_bench_c5.log 2>&1
python bench.py --config 4 --no-e2e > gpurun_out/b6_bench_c4.log 2>&1
python bench.py --config 2 > gpurun_out/b6_bench_c2.log 2>&1
python bench.py --config 1 > gpurun_out/b6_bench_c1.log 2>&1
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b6_launches.csv python bench.py --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/b6_ncu_launches.log 2>&1
python scripts/diag.py --config 3 > gpurun_out/b6_diag_c3.log 2>&1
python scripts/diag.py --config 4 > gpurun_out/b6_diag_c4.log 2>&1
python scripts/diag.py --config 5 --iters 5 > gpurun_out/b6_diag_c5.log 2>&1
SSLIC_TIMING=1 python bench.py --config 3 --no-cpu > gpurun_out/b6_e2e_c3.log 2> gpurun_out/b6_e2e_c3.err
