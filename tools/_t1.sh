set -u
mkdir -p gpurun_out
M=gpu__time_duration.sum
ncu --metrics $M --clock-control none -k 'regex:k_cell_res|k_cell_pa|k_face_pa8' --csv --log-file gpurun_out/ab_pf3.csv python tools/prof_solve.py C5 256 2 > /dev/null 2>&1
grep -h "k_cell_res\|k_cell_pa\|k_face_pa8" gpurun_out/ab_pf3.csv | awk -F'","' '{if ($NF+0 > 12000) printf "%s:%s ", substr($5,16,12), $NF} END {print ""}'
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_zero_first.py -x -q 2>&1 | tail -2
for i in 1 2; do python bench.py --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C5', d['value'], d['clocks']['sm_mhz'])"; done
python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C4', d['value'], d['clocks']['sm_mhz'])"
