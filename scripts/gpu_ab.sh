# A/B: per-iteration diagnostics with the in-tree library and libsslic_b200_ab.so, alternating
cd $GRAFT_REPO_ROOT
T=${1:-ab}; C=${2:-3}
for r in 1 2; do
  python scripts/diag.py --config $C > gpurun_out/${T}_new$r.log 2>&1
  SSLIC_B200_LIB=$PWD/paper_1806_08741_b200/libsslic_b200_ab.so python scripts/diag.py --config $C > gpurun_out/${T}_ab$r.log 2>&1
done
