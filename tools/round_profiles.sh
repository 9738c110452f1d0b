#!/bin/bash
# The round's measurement set (run under gpurun, one GPU):
#   bench line (+ e2e), reference arm, launch list of one full solve, and an
#   ncu --set full capture of the finest-level face colour passes and the
#   Arnoldi passes.  Each ncu run follows the same command without ncu.
set -u
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
echo "bench rc=$?"
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
echo "reference rc=$?"
bash tools/prof_full.sh
python tools/prof_kernels.py C5 256 > gpurun_out/pk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_face_colour -c 3 \
    -o gpurun_out/final_face_colour python tools/prof_kernels.py C5 256 > gpurun_out/ncu_fc.log 2>&1
echo "ncu face colour rc=$?"
python tools/prof_solve.py C5 256 20 > gpurun_out/ps_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_dcgs -s 30 -c 2 \
    -o gpurun_out/final_dcgs python tools/prof_solve.py C5 256 20 > gpurun_out/ncu_dcgs.log 2>&1
echo "ncu dcgs rc=$?"
# Summarise on the box (the .ncu-rep files are too large to bring back) and
# keep only the summaries + the launch list in gpurun_out/.
for r in final_face_colour final_dcgs; do
  [ -f gpurun_out/$r.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.json && \
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
  mv -f gpurun_out/$r.ncu-rep /tmp/ 2>/dev/null
done
python tools/launch_summary.py gpurun_out/launches_full.csv > gpurun_out/launch_summary.txt 2>&1
du -sh gpurun_out
