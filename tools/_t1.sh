set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in C5 C4 C3; do
python bench.py --config $c --no-cpu-baseline --steps 3 > gpurun_out/b_$c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', d['value'], d['e2e']['value'], d['roofline']['frac'], {k:round(v,3) for k,v in d['smoother'].items() if 'frac' in k}, d['clocks']['sm_mhz'])"
done
