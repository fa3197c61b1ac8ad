cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_heat_gpu.py -q -m gpu -x -k "dst" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
python tools/profile_heat.py --nt 64 > gpurun_out/plain_heat.log 2>&1; cat gpurun_out/plain_heat.log
python tools/profile_heat.py --nt 64 --transform dst > gpurun_out/plain_heat_dst.log 2>&1; cat gpurun_out/plain_heat_dst.log
