cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ntt_fwd_rows -s 2 -c 1 -o gpurun_out/ntt_rows python tools/ntt_prof.py > gpurun_out/ntt_prof.log 2>&1
