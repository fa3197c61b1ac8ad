cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench rc=$?; cat gpurun_out/bench.log; tail -3 gpurun_out/bench.err
