cd $GRAFT_REPO_ROOT
T=${1:-misc}
timeout 1500 python -m pytest tests -m gpu -q -x -k "not test_config_matches_reference" > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
bash scripts/ab.sh ${T}_c1 "X=0" "SSLIC_NO_SMALL_UPDATE=1" --config 1 > gpurun_out/${T}_ab_c1.txt 2>&1
bash scripts/ab.sh ${T}_c2 "X=0" "SSLIC_NO_SMALL_UPDATE=1" --config 2 > gpurun_out/${T}_ab_c2.txt 2>&1
