#!/bin/bash
# run scripts/gpu_run15.sh with a tag and summarize
TAG=$1
/usr/local/graft/bin/gpurun --timeout 1500 -- "bash scripts/gpu_run15.sh $TAG" > /tmp/gpurun_$TAG.out 2>&1
tail -1 /tmp/gpurun_$TAG.out
tail -2 gpurun_out/${TAG}_pytest.log
for c in c3 c4 c5; do tail -2 gpurun_out/${TAG}_$c.log | head -1; done
