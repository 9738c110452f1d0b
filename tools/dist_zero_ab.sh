# A/B of the slab path's zero fills: one k_zero_segs launch vs a memset per range
mkdir -p gpurun_out
for m in 0 1 0 1; do
  SB_DIST_ZERO_MEMSET=$m timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port $((29620 + RANDOM % 100)) bench.py --gpus 1 --force-dist --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SB_DIST_ZERO_MEMSET=$m', round(d['value'],4), d['clocks']['sm_mhz'])"
done
