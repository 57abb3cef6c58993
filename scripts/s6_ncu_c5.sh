# per-source-line instruction profile of the config-5 lean kernel (one launch, iteration 3)
cd $GRAFT_REPO_ROOT
T=${1:-s6}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_assign_lean -s 6 -c 1 -o /tmp/${T}_c5 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_c5.log 2>&1
python scripts/ncu_summary.py /tmp/${T}_c5.ncu-rep > gpurun_out/${T}_c5_summary.txt 2>&1
python scripts/ncu_lines.py /tmp/${T}_c5.ncu-rep 400 > gpurun_out/${T}_c5_lines.txt 2>&1
python scripts/ncu_regions.py /tmp/${T}_c5.ncu-rep > gpurun_out/${T}_c5_regions.txt 2>&1
