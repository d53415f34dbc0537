# compute-sanitizer on the smoke sequence (toy PCMM, ring packing, SlotToCoeffs): memcheck (out-of-bounds /
# misaligned accesses), racecheck (shared-memory hazards), initcheck (reads of uninitialized device memory)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for tool in memcheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/smoke_repro.py 1 > gpurun_out/san_$tool.txt 2>&1
  echo "$tool exit $?" >> gpurun_out/san_$tool.txt
done
