cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_bench.log 2>&1 && \
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
python tools/profile_heat.py --nt 64 > gpurun_out/plain_heat.log 2>&1 && \
$NCU --set full --clock-control none --import-source on -k regex:gemm_f64 -s 0 -c 2 -o gpurun_out/prof_gemm_heat_v2 python tools/profile_heat.py --nt 64 > gpurun_out/ncu_gemm.log 2>&1; echo gemm rc=$?
python tools/profile_wave.py 5 > gpurun_out/plain_wave.log 2>&1 && \
$NCU --set full --clock-control none -k regex:"gemm_f64|wave_apply|gemv|dot_partials|cg_update" -s 0 -c 12 -o gpurun_out/prof_wave_v2 python tools/profile_wave.py 5 > gpurun_out/ncu_wave.log 2>&1; echo wave rc=$?
