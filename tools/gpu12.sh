cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_wave_gpu.py -q -m gpu -x -s -k cfg4 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; grep -E "cfg4|passed|failed|Error" gpurun_out/pytest_gpu.log | tail -8
