cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for cfg in "32 0" "16 0" "8 0" "32 1" "16 1" "8 1"; do
  set -- $cfg
  export HE_MS_JC=$1
  if [ $2 = 1 ]; then export HE_RP_INTERLEAVE=1; else unset HE_RP_INTERLEAVE; fi
  echo "JC=$1 INTERLEAVE=$2: $(python tools/ringpack_kernel_times.py 2>/dev/null | head -1)"
done > gpurun_out/rp_jc.txt 2>&1
