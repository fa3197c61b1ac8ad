cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_wave_gpu.py tests/test_cpp_api.py -q -m gpu -x -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; grep -E "cfg4|passed|failed|Error" gpurun_out/pytest_gpu.log | tail -8
python tools/profile_wave.py 40 > gpurun_out/plain_wave.log 2>&1 && \
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_wave.csv python tools/profile_wave.py 40 > gpurun_out/ncu_wave.log 2>&1; echo ncu rc=$?
