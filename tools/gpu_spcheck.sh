# full-output parity vs the CPU spectral restatement (all Llama shapes) + the bench line with the new cpu_baseline
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
make -s -C oracle
timeout 1200 python -m pytest tests/test_gpu_pcmm.py -x -q -k "full_output" --durations=10 > gpurun_out/pytest_spcheck.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_spcheck.log
timeout 600 python bench.py --no-extras > gpurun_out/bench_sp.json 2> gpurun_out/bench_sp.err; echo "bench exit $?" >> gpurun_out/bench_sp.err
