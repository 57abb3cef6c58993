cd $GRAFT_REPO_ROOT
T=${1:-p16}
python bench.py --config 3 --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 9 -c 1 -o gpurun_out/${T}_assign_c3 python bench.py --config 3 --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_c3_ncu.log 2>&1
echo "rc $?" >> gpurun_out/${T}_c3_ncu.log
