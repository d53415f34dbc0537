# ncu evidence for profiles/r02: the bench launch list and one --set full capture of every spectral-path kernel
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 1 --cpu-rows 0 --no-e2e --no-extras --no-direct > gpurun_out/ncu_launch_bench.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spec_|modgemm2|decompose" -s 7 -c 7 -o gpurun_out/prof_spectral_r02 python tools/profile_op.py --ops 2 > gpurun_out/ncu_spectral.out 2>&1
python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
