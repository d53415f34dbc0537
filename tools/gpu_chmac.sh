cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none -k regex:k_ch_mac -s 2 -c 1 -o gpurun_out/chmac python tools/chain_times.py 6 > gpurun_out/chmac.log 2>&1
