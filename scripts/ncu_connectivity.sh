# ncu --set full captures of the connectivity kernels on config 3
# (scripts/conn_time.py --config 3 --no-ref --reps 1), one launch each,
# summarised on the box (scripts/ncu_summary.py).
cd $GRAFT_REPO_ROOT
T=${1:-nccc}
for k in k_cc_tile k_cc_seams k_edge_list k_edges_list; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:^$k\$ -c 1 \
    -o /tmp/${T}_$k python scripts/conn_time.py --config 3 --no-ref --reps 1 \
    > gpurun_out/${T}_ncu_$k.log 2>&1
  python scripts/ncu_summary.py /tmp/${T}_$k.ncu-rep > gpurun_out/${T}_${k}_summary.txt 2>&1
done
head -16 gpurun_out/${T}_k_cc_seams_summary.txt
