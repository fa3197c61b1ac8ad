#!/bin/bash
# Full GPU check: pytest -m gpu, smoke, default bench line, cfg5 padded-layout A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; tail -c 300 gpurun_out/bench.log
for pad in 1 0; do echo "cfg5 PAD=$pad"; STKG_PAD=$pad python tools/profile_cfg5.py 2>&1 | tail -2; done
