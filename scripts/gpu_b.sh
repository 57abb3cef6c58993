# bench lines: config 3 with phase timing, plus optional configs
cd $GRAFT_REPO_ROOT
TAG=${1:-b}
shift
SSLIC_TIMING=1 python bench.py --config 3 --no-cpu > gpurun_out/${TAG}_b3.log 2> gpurun_out/${TAG}_b3.err
for c in $@; do python bench.py --config $c --no-cpu > gpurun_out/${TAG}_b$c.log 2>&1; done
