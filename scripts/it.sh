# local helper: run scripts/gpu_it.sh on the GPU box and print a summary
TAG=$1; shift
/usr/local/graft/bin/gpurun --timeout 1500 -- "bash scripts/gpu_it.sh $TAG $*" > /tmp/gpurun_$TAG.out 2>&1
tail -1 /tmp/gpurun_$TAG.out; tail -2 gpurun_out/${TAG}_pytest.log | head -1
for f in gpurun_out/${TAG}_c*.log; do echo $f; grep "^iter" $f | cut -c1-44 | tr '\n' ' ' | sed 's/assign//g'; echo; done
