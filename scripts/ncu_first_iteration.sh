# ncu --set full of config 3's first-iteration kernel (launch 3 of bench.py --warmup 3 = iteration 0 of the first timed run)
cd $GRAFT_REPO_ROOT
T=${1:-first}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 3 -c 1 -o /tmp/${T}_c3 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_c3.log 2>&1
python scripts/ncu_summary.py /tmp/${T}_c3.ncu-rep > gpurun_out/${T}_c3_summary.txt 2>&1
python scripts/ncu_lines.py /tmp/${T}_c3.ncu-rep 400 > gpurun_out/${T}_c3_lines.txt 2>&1
python scripts/ncu_regions.py /tmp/${T}_c3.ncu-rep > gpurun_out/${T}_c3_regions.txt 2>&1
