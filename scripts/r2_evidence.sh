# round-2 evidence, part 1: the config-3 bench (driver's K/W), the other
# configs, the N>1 code path at N=1, and the reference arm
cd $GRAFT_REPO_ROOT
T=${1:-ev}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${T}_smi.txt 2>&1
SSLIC_TIMING=1 timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_c3.log 2> gpurun_out/${T}_bench_c3.err
for c in 1 2 4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${T}_bench_c$c.log 2>&1; done
timeout 1200 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e > gpurun_out/${T}_bench_c5.log 2>&1
timeout 900 python bench.py --nccl --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_bench_c3_nccl.log 2>&1
if [ "${REF:-1}" = 1 ]; then
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_ref_c3.log 2>&1
fi
