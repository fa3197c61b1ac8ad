cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench.log 2>&1; echo bench rc=$?; cat gpurun_out/bench.log
python tools/profile_heat.py --nt 64 > gpurun_out/plain_heat.log 2>&1 && \
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:heat_apply -s 0 -c 1 -o gpurun_out/prof_apply_v2 python tools/profile_heat.py --nt 64 > gpurun_out/ncu_apply.log 2>&1; echo apply rc=$?
