# ncu --set full capture of config 5's assign kernel (last timed iteration)
cd $GRAFT_REPO_ROOT
T=${1:-p5}
python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_c5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 4 -c 1 -o gpurun_out/${T}_assign_c5 python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_c5_ncu.log 2>&1
echo "rc $?" >> gpurun_out/${T}_c5_ncu.log
