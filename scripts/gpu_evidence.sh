# round evidence: GPU tests, smoke, bench lines (configs 1-5 + reference arm),
# launch list, ncu captures of the assign kernel, per-iteration diagnostics
cd $GRAFT_REPO_ROOT
T=${1:-ev}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${T}_smoke.log
SSLIC_TIMING=1 python bench.py > gpurun_out/${T}_bench_c3.log 2> gpurun_out/${T}_bench_c3.err
python bench.py --impl reference > gpurun_out/${T}_ref_c3.log 2>&1
python bench.py --config 1 > gpurun_out/${T}_bench_c1.log 2>&1
python bench.py --config 2 > gpurun_out/${T}_bench_c2.log 2>&1
python bench.py --config 4 > gpurun_out/${T}_bench_c4.log 2>&1
python bench.py --config 5 --steps 2 --warmup 3 --no-e2e > gpurun_out/${T}_bench_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c3.csv python bench.py --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 9 -c 1 -o gpurun_out/${T}_assign_c3 python bench.py --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 9 -c 1 -o gpurun_out/${T}_assign_c4 python bench.py --config 4 --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_c4.log 2>&1
python scripts/diag.py --config 3 > gpurun_out/${T}_diag_c3.log 2>&1
python scripts/diag.py --config 4 > gpurun_out/${T}_diag_c4.log 2>&1
python scripts/diag.py --config 5 --iters 5 > gpurun_out/${T}_diag_c5.log 2>&1
