cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_pcmm.py -x -q -k "llama_ring_keygen" > gpurun_out/pytest_enc.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_enc.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --dist-backend gloo --one-device --steps 2 --warmup 1 --no-e2e > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; echo "exit $?" >> gpurun_out/bench_2rank.err
