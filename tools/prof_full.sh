#!/bin/bash
# launch list of one FULL C5 256^3 P1 solve, for per-kernel shares
python tools/prof_solve.py C5 256 500 > gpurun_out/plain_full.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_full.csv \
    python tools/prof_solve.py C5 256 500 > gpurun_out/ncu_full.log 2>&1
echo "full launch list rc=$?"
