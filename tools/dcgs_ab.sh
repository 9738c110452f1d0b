#!/bin/bash
# A/B of the Arnoldi pass-A kernels (SB_DCGS_A) on the C5 256^3 bench solve,
# then ncu launch times of pass A per variant.
set -u
for v in 2 32 34 24 323 343; do
  SB_DCGS_A=$v python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/ab_dcgs_$v.json 2> gpurun_out/ab_dcgs_$v.err
  echo "variant $v rc=$? $(python -c "import json;d=json.load(open('gpurun_out/ab_dcgs_$v.json'));print(d['value'],d['config']['iterations'])")"
done
python tools/prof_solve.py C5 256 20 > /dev/null 2>&1
for v in 2 32 34 323 343; do
  SB_DCGS_A=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:k_dcgs_a --csv --log-file gpurun_out/ab_dcgs_ncu_$v.csv python tools/prof_solve.py C5 256 20 > /dev/null 2>&1
  echo "ncu $v rc=$?"
done
