# round-1 second-half evidence: bench line, its launch list, --set full of S3/S4, ring packing and slot PCMM kernels
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_v12.json 2> gpurun_out/bench_v12.err; echo "bench exit $?" >> gpurun_out/bench_v12.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v12.csv python bench.py --steps 2 --warmup 1 --cpu-rows 0 --no-e2e --no-extras --no-direct > gpurun_out/ncu_launch_v12.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spec_gemm|spec_inverse" -s 5 -c 3 -o gpurun_out/prof_spectral_v4 python tools/profile_op.py --ops 2 > gpurun_out/ncu_spectral_v4.out 2>&1
timeout 600 ncu --set full --clock-control none --profile-from-start off -k regex:"k_ms_|ntt_fwd" -c 6 -o gpurun_out/prof_ringpack python tools/ringpack_prof.py > gpurun_out/ncu_ringpack.out 2>&1
timeout 600 ncu --set full --clock-control none --profile-from-start off -k regex:"k_sd_|ntt_" -c 12 -o gpurun_out/prof_slotpcmm python tools/slotpcmm_prof.py > gpurun_out/ncu_slotpcmm.out 2>&1
ls -la gpurun_out
