#!/bin/bash
# Round profile capture at C5 (one B200): launch list of one step, then one
# `ncu --set full` capture per listing kernel (separate ncu sessions).
# At C5 class H runs the CTA-wide kernel, so k_list_cta launches are H, C1, C2.
#   tools/profile_c5.sh <tag>
TAG=${1:-r02c}; CFG=c5
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
prof() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 \
      -o gpurun_out/prof_${TAG}_$1 $CMD > gpurun_out/ncu_full_${TAG}_$1.log 2>&1
}
prof reg k_list_reg 0
prof cta_h k_list_cta 0
prof cta_c1 k_list_cta 1
prof cta_c2 k_list_cta 2
for k in reg cta_h cta_c1 cta_c2; do
  R=gpurun_out/prof_${TAG}_$k.ncu-rep
  [ -f "$R" ] || continue
  ncu -i $R --page raw --csv > gpurun_out/raw_${TAG}_$k.csv 2>/dev/null
  ncu -i $R --page source --csv > /tmp/src_$k.csv 2>/dev/null && python tools/ncu_src.py /tmp/src_$k.csv 0.004 > gpurun_out/src_${TAG}_$k.txt 2>&1
  ncu -i $R --page source --print-source cuda,sass --csv > gpurun_out/srccuda_${TAG}_$k.csv 2>/dev/null
  gzip -f gpurun_out/srccuda_${TAG}_$k.csv
  rm -f $R
done
echo "profile_c5 done"
