cd $GRAFT_REPO_ROOT
python tools/profile_heat.py --nt 64 --transform dst > gpurun_out/plain_heat_dst.log 2>&1 && \
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:dst_axis -s 0 -c 2 -o gpurun_out/prof_dst python tools/profile_heat.py --nt 64 --transform dst > gpurun_out/ncu_dst.log 2>&1; echo ncu rc=$?
