cd $GRAFT_REPO_ROOT
python bench.py --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/p16_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 9 -c 1 -o gpurun_out/p16_assign python bench.py --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/p16_ncu.log 2>&1
echo "rc $?" >> gpurun_out/p16_ncu.log
