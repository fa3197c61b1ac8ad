cd $GRAFT_REPO_ROOT
python tools/profile_heat.py --nt 1024 --transform dst --reps 1 > gpurun_out/plain_heat_dst.log 2>&1 && cat gpurun_out/plain_heat_dst.log && \
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --csv --log-file gpurun_out/launches_dst.csv python tools/profile_heat.py --nt 1024 --transform dst --reps 1 > gpurun_out/ncu_l.log 2>&1; echo rc=$?
