cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none -k regex:"k_ch_combine|k_ch_inner|k_ch_lift|k_ch_digits" -s 4 -c 4 -o gpurun_out/chmac python tools/chain_times.py 6 > gpurun_out/chmac.log 2>&1
