# full GPU suite + smoke (round evidence)
cd $GRAFT_REPO_ROOT
T=${1:-full}
rm -f gpurun_out/reference_configs.jsonl
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
cp gpurun_out/reference_configs.jsonl gpurun_out/${T}_reference_configs.jsonl 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${T}_smoke.log
