# A/B of the one-CTA coarse tail start (SB_COARSE_CELLS) on C5 / C3, same box
mkdir -p gpurun_out
for c in 512 64 512 64; do
  SB_COARSE_CELLS=$c python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 SB_COARSE_CELLS=$c', round(d['value'],4), d['clocks']['sm_mhz'])"
done
for c in 512 64; do
  SB_COARSE_CELLS=$c python bench.py --config C3 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 SB_COARSE_CELLS=$c', round(d['value'],5))"
done
