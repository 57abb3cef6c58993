# per-source-line instruction profile of the config-3 assign kernel (one launch, iteration 5)
cd $GRAFT_REPO_ROOT
T=${1:-lines}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 8 -c 1 -o /tmp/${T}_c3 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_c3.log 2>&1
python scripts/ncu_summary.py /tmp/${T}_c3.ncu-rep > gpurun_out/${T}_c3_summary.txt 2>&1
python scripts/ncu_lines.py /tmp/${T}_c3.ncu-rep 400 > gpurun_out/${T}_c3_lines.txt 2>&1
python scripts/ncu_regions.py /tmp/${T}_c3.ncu-rep > gpurun_out/${T}_c3_regions.txt 2>&1
T=${1:-lines}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_assign_lean -s 6 -c 1 -o /tmp/${T}_c5 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_c5.log 2>&1
python scripts/ncu_summary.py /tmp/${T}_c5.ncu-rep > gpurun_out/${T}_c5_summary.txt 2>&1
python scripts/ncu_lines.py /tmp/${T}_c5.ncu-rep 400 > gpurun_out/${T}_c5_lines.txt 2>&1
python scripts/ncu_regions.py /tmp/${T}_c5.ncu-rep > gpurun_out/${T}_c5_regions.txt 2>&1
