# A/B of the face colour row mapping (SB_FC_BX / SB_FC_BX_MIN) on the C5 bench, same box
mkdir -p gpurun_out
for m in 0 128 0 128; do
  SB_FC_BX_MIN=$m python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SB_FC_BX_MIN=$m', round(d['value'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
for m in 0 128; do
  SB_FC_BX_MIN=$m python bench.py --config C3 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 SB_FC_BX_MIN=$m', round(d['value'],5))"
done
