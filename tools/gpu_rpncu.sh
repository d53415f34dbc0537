cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ms1_digits_cols|k_ms1_mac_y" -s 2 -c 2 -o gpurun_out/rpk python tools/ringpack_prof.py --method keyswitch1 > gpurun_out/rpk.log 2>&1
python tools/ncu_summary.py gpurun_out/rpk.ncu-rep --source "ncu --set full tools/ringpack_prof.py --method keyswitch1" -o gpurun_out/rpk_summary.json >> gpurun_out/rpk.log 2>&1
