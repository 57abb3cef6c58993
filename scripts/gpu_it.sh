# iterate: GPU tests, then per-iteration diagnostics for the given configs (default 3 4)
cd $GRAFT_REPO_ROOT
TAG=${1:-x}
shift
CFGS=${@:-3 4}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
for c in $CFGS; do
  if [ $c = 5 ]; then python scripts/diag.py --config 5 --iters 5 > gpurun_out/${TAG}_c5.log 2>&1
  else python scripts/diag.py --config $c > gpurun_out/${TAG}_c$c.log 2>&1; fi
done
