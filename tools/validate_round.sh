mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --force-dist --steps 3 --warmup 3 > gpurun_out/slab1.json 2> gpurun_out/slab1.err; echo "slab1 rc=$?"
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4.json 2> gpurun_out/c4.err; echo "c4 rc=$?"
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c3.json 2> gpurun_out/c3.err; echo "c3 rc=$?"
timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c2.json 2> gpurun_out/c2.err; echo "c2 rc=$?"
