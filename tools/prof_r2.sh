#!/bin/bash
# Round-2 profiling set (one GPU): C4 256^3 launch list (30 iterations), ncu
# --set full of the row-vector apply_M / residual kernels (C5) and of the walled
# finest-level colour passes (C4).  Each ncu run follows the same command
# without ncu; reports are summarised on the box (too large to bring back).
set -u
mkdir -p gpurun_out
python tools/prof_solve.py C4 256 30 > gpurun_out/c4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
    python tools/prof_solve.py C4 256 30 > gpurun_out/ncu_c4.log 2>&1
echo "c4 launch list rc=$?"
python tools/launch_summary.py gpurun_out/launches_c4.csv > gpurun_out/launch_summary_c4.txt 2>&1
python tools/prof_kernels.py C5 256 > gpurun_out/pk5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_face_all_rv -c 2 \
    -o gpurun_out/r02_face_all_rv python tools/prof_kernels.py C5 256 > gpurun_out/ncu_rv.log 2>&1
echo "ncu rv rc=$?"
python tools/prof_kernels.py C4 256 > gpurun_out/pk4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k 'regex:k_face_colour|k_cell_colour|k_apply_M|k_face_res' -c 12 \
    -o gpurun_out/r02_c4_colour python tools/prof_kernels.py C4 256 > gpurun_out/ncu_c4c.log 2>&1
echo "ncu c4 colour rc=$?"
for r in r02_face_all_rv r02_c4_colour; do
  [ -f gpurun_out/$r.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.json && \
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
  ls -la gpurun_out/$r.ncu-rep
  mv -f gpurun_out/$r.ncu-rep /tmp/ 2>/dev/null
done
du -sh gpurun_out
