cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x -k "cfg3 or cfg4" -s > gpurun_out/pytest_big.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_big.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.log; tail -5 gpurun_out/bench.err
