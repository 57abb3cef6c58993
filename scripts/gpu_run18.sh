cd $GRAFT_REPO_ROOT
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
SSLIC_TIMING=1 python bench.py --config 3 --no-cpu > gpurun_out/${TAG}_b3.log 2> gpurun_out/${TAG}_b3.err
SSLIC_TIMING=1 python bench.py --config 2 --no-cpu > gpurun_out/${TAG}_b2.log 2> gpurun_out/${TAG}_b2.err
