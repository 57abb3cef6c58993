cd $GRAFT_REPO_ROOT
T=${1:-t}
shift
timeout 1500 python -m pytest "$@" -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
