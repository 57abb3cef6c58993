cd $GRAFT_REPO_ROOT
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
python scripts/diag.py --config 3 > gpurun_out/${TAG}_c3.log 2>&1
python scripts/diag.py --config 4 > gpurun_out/${TAG}_c4.log 2>&1
python scripts/diag.py --config 5 --iters 4 > gpurun_out/${TAG}_c5.log 2>&1
