# round-2 evidence: GPU tests, smoke, config-3 bench (driver's K/W), the
# reference arm, the launch list and one ncu --set full of the assign kernel
cd $GRAFT_REPO_ROOT
T=${1:-ev}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${T}_smi.txt 2>&1
nproc > gpurun_out/${T}_host.txt; free -g >> gpurun_out/${T}_host.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_c3.log 2> gpurun_out/${T}_bench_c3.err
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c3.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 9 -c 1 -o gpurun_out/${T}_assign_c3 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_c3.log 2>&1
fi
if [ "${REF:-1}" = 1 ]; then
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_ref_c3.log 2>&1
fi
