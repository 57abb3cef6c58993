cd $GRAFT_REPO_ROOT
T=${1:-rest}
timeout 1200 python -m pytest tests/test_gpu_reference_configs.py tests/test_gpu_synth.py tests/test_io_volumes.py tests/test_multi.py -m gpu -q -k "not test_config_matches_reference" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
cp gpurun_out/reference_configs.jsonl gpurun_out/${T}_reference_configs.jsonl 2>/dev/null
timeout 600 python bench.py --nccl --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_bench_nccl.log 2>&1
bash scripts/r2_conn.sh ${T}conn
