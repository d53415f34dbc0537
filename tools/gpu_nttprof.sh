cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ntt_(fwd|inv)_(rows|cols)" -s 4 -c 4 -o gpurun_out/ntt_rows python tools/ntt_prof.py > gpurun_out/ntt_prof.log 2>&1
python tools/ncu_summary.py gpurun_out/ntt_rows.ncu-rep --source "ncu --set full tools/ntt_prof.py" -o gpurun_out/ntt_rows_summary.json >> gpurun_out/ntt_prof.log 2>&1
