cd $GRAFT_REPO_ROOT
python bench.py --config 4 --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/p15_c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 9 -c 1 -o gpurun_out/p15_assign_c4 python bench.py --config 4 --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/p15_c4_ncu.log 2>&1
echo "rc $?" >> gpurun_out/p15_c4_ncu.log
python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p15_c5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 4 -c 1 -o gpurun_out/p15_assign_c5 python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p15_c5_ncu.log 2>&1
echo "rc $?" >> gpurun_out/p15_c5_ncu.log
