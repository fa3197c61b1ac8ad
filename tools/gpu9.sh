cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_heat_gpu.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench.log 2>&1; echo bench rc=$?; python -c "import json; d=json.load(open('gpurun_out/bench.log')); print(d['k1_residual'], d['k3_scan'])"
