#!/bin/bash
# baselines of the secondary configs + ncu source-level capture of the H and C1 kernels (C4, count+checksum)
bash tools/r02_run4.sh
CMD="python tools/ab.py --config c4 --flags 1 --reps 1 --libs _cks0"
$CMD > gpurun_out/plain5.log 2>&1 || exit 1
for k in warp cta; do
  ncu --set full --clock-control none --import-source on -k regex:k_list_$k -s 1 -c 1 -o gpurun_out/prof5_$k $CMD > gpurun_out/ncu5_$k.log 2>&1
  ncu -i gpurun_out/prof5_$k.ncu-rep --page raw --csv > gpurun_out/raw5_$k.csv 2>/dev/null
  ncu -i gpurun_out/prof5_$k.ncu-rep --page source --csv > gpurun_out/src5_$k.csv 2>/dev/null
  ncu -i gpurun_out/prof5_$k.ncu-rep --page details --csv > gpurun_out/det5_$k.csv 2>/dev/null
  rm -f gpurun_out/prof5_$k.ncu-rep
done
ls -la gpurun_out/
