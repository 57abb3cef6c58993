cd $GRAFT_REPO_ROOT
python bench.py --config 2 --path exact --no-cpu --no-e2e > gpurun_out/ex_c2.log 2>&1
python bench.py --config 4 --path exact --no-cpu --no-e2e > gpurun_out/ex_c4.log 2>&1
python bench.py --config 3 --path exact --no-cpu --no-e2e --steps 3 > gpurun_out/ex_c3.log 2>&1
