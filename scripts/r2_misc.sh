cd $GRAFT_REPO_ROOT
T=${1:-misc}
bash scripts/ab.sh ${T}_dyn "X=0" "SSLIC_DYN=1" > gpurun_out/${T}_ab_dyn.txt 2>&1
SSLIC_DYN=1 timeout 1200 python -m pytest tests/test_gpu_fast.py tests/test_gpu_fullsize.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
