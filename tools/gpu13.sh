cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_heat_gpu.py -q -m gpu -x -k "dst" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -30 gpurun_out/pytest_gpu.log
