cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r14_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r14_pytest.log
python scripts/diag.py --config 3 > gpurun_out/d10_c3.log 2>&1
python scripts/diag.py --config 4 > gpurun_out/d10_c4.log 2>&1
python scripts/diag.py --config 5 --iters 4 > gpurun_out/d10_c5.log 2>&1
python scripts/diag.py --config 2 > gpurun_out/d10_c2.log 2>&1
python bench.py --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/p10_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_assign_fast -s 9 -c 1 -o gpurun_out/p10_assign python bench.py --steps 7 --warmup 3 --no-e2e --no-cpu > gpurun_out/p10_ncu.log 2>&1
