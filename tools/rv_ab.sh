#!/bin/bash
# A/B of the finest-level face kernels (ncu launch times + DRAM bytes):
#   base = per-face kernels with stored mu_e, de = per-face with derived mu_e,
#   rv3/rv4 = row-vector kernels (derived mu_e) compiled for 3 / 4 CTAs per SM
set -u
python tools/prof_kernels.py C5 256 > gpurun_out/pk.log 2>&1; echo pk rc=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
K='regex:rv|k_face_colour|k_apply_M|k_face_res'
run() { env "$@" ncu --metrics $M --clock-control none -k "$K" --csv --log-file gpurun_out/ab_$1.csv python tools/prof_kernels.py C5 256 > /dev/null 2>&1; echo "$1 rc=$?"; }
run_named() { local name=$1; shift; env "$@" ncu --metrics $M --clock-control none -k "$K" --csv --log-file gpurun_out/ab_$name.csv python tools/prof_kernels.py C5 256 > /dev/null 2>&1; echo "$name rc=$?"; }
run_named base SB_ROWV=0 SB_MUE_DERIVED=0
run_named de SB_ROWV=0
run_named rv3 SB_ROWV_MINB=3
run_named rv4 SB_ROWV_MINB=4
run_named rvnode SB_ROWV_MINB=4 SB_MUE_DERIVED=0
