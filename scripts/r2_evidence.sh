# round-2 evidence: config-3 bench (driver's K/W), the other configs, the
# reference arm, the launch list and ncu --set full captures of the assign
# kernels (config 3: k_assign_fast, config 5: k_assign_lean)
cd $GRAFT_REPO_ROOT
T=${1:-ev}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${T}_smi.txt 2>&1
SSLIC_TIMING=1 timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_c3.log 2> gpurun_out/${T}_bench_c3.err
for c in 1 2 4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${T}_bench_c$c.log 2>&1; done
timeout 1200 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/${T}_bench_c5.log 2>&1
timeout 900 python bench.py --nccl --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_bench_c3_nccl.log 2>&1
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c3.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 9 -c 1 -o gpurun_out/${T}_assign_c3 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assign_lean -s 4 -c 1 -o gpurun_out/${T}_lean_c5 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 9 -c 1 -o gpurun_out/${T}_assign_c4 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_c4.log 2>&1
fi
if [ "${REF:-1}" = 1 ]; then
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_ref_c3.log 2>&1
fi
