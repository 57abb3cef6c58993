cd $GRAFT_REPO_ROOT
SSLIC_BENCH_FUNCTIONAL_CHECK=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config 4 --steps 2 --warmup 3 > gpurun_out/func_n2.log 2>&1
echo "rc $?" >> gpurun_out/func_n2.log
