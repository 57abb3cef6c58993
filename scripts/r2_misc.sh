cd $GRAFT_REPO_ROOT
T=${1:-misc}
timeout 1200 python -m pytest tests/test_gpu_fast.py tests/test_gpu_fullsize.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
bash scripts/ab.sh ${T}_tma "X=0" "SSLIC_NO_TMA=1" > gpurun_out/${T}_ab_tma.txt 2>&1
