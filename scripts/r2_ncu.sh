# round-2 evidence, part 2: launch list + ncu --set full captures of the
# assign kernels, summarised on the box (reports are large: only the
# config-3 one is kept)
cd $GRAFT_REPO_ROOT
T=${1:-ncu}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c3.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_launches.log 2>&1
cap() {  # name kernel-regex skip bench-args...
  local name=$1 kern=$2 skip=$3; shift 3
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$kern -s $skip -c 1 -o /tmp/${T}_$name python bench.py "$@" --no-e2e --no-cpu > gpurun_out/${T}_ncu_$name.log 2>&1
  python scripts/ncu_summary.py /tmp/${T}_$name.ncu-rep > gpurun_out/${T}_${name}_summary.txt 2>&1
}
cap assign_c3 k_assign_fast 9 --steps 10 --warmup 3
python scripts/ncu_sass.py /tmp/${T}_assign_c3.ncu-rep --top 40 > gpurun_out/${T}_assign_c3_sass.txt 2>&1
cp /tmp/${T}_assign_c3.ncu-rep gpurun_out/ 2>/dev/null
cap lean_c5 k_assign_lean 4 --config 5 --steps 5 --warmup 3
cap assign_c4 k_assign_fast 9 --config 4 --steps 10 --warmup 3
ls -la gpurun_out/ > gpurun_out/${T}_ls.txt
