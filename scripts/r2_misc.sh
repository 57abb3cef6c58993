cd $GRAFT_REPO_ROOT
T=${1:-misc}
bash scripts/ab.sh ${T}_full "X=0" "SSLIC_NO_FULL=1" > gpurun_out/${T}_ab_full.txt 2>&1
timeout 900 python bench.py --nccl --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_bench_c3_nccl.log 2>&1
timeout 1200 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e > gpurun_out/${T}_bench_c5.log 2>&1
