cd $GRAFT_REPO_ROOT
T=${1:-misc}
bash scripts/ab.sh ${T}_six "X=0" "SSLIC_SIX=1" > gpurun_out/${T}_ab_six.txt 2>&1
SSLIC_SIX=1 timeout 1200 python -m pytest tests/test_gpu_fast.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
