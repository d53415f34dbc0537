cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/rp_launches.csv python tools/ringpack_prof.py --method keyswitch1 > gpurun_out/rp_prof.log 2>&1
