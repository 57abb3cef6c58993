cd $GRAFT_REPO_ROOT
TAG=${1:-v2}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench_c3.log 2>&1
python scripts/diag.py --config 3 > gpurun_out/${TAG}_diag_c3.log 2>&1
