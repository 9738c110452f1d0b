set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
bash tools/validate_round.sh
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 1 --force-dist --config C4 --steps 2 --warmup 2 > gpurun_out/slab1_c4.json 2> gpurun_out/slab1_c4.err; echo "slab1 c4 rc=$?"
timeout 1500 bash tools/round_profiles.sh
