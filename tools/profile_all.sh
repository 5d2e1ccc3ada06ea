#!/bin/bash
# Round profile capture (one B200): launch list of one C4 step, then one
# `ncu --set full` capture per listing kernel, each in its own ncu session (a
# second kernel captured in one session came back with empty metrics).
#   tools/profile_all.sh <tag> [config]
TAG=${1:-r01}; CFG=${2:-c4}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
prof() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 \
      -o gpurun_out/prof_${TAG}_$1 $CMD > gpurun_out/ncu_full_${TAG}_$1.log 2>&1
}
prof reg k_list_reg 0
prof warp k_list_warp 0
prof cta_c1 k_list_cta 0
prof cta_c2 k_list_cta 1
echo "profile_all done"
# export summaries on the box and drop the big .ncu-rep files (gpurun brings
# back at most 64 MiB of gpurun_out/)
for k in reg warp cta_c1 cta_c2; do
  R=gpurun_out/prof_${TAG}_$k.ncu-rep
  [ -f "$R" ] || continue
  ncu -i $R --page raw --csv > gpurun_out/raw_${TAG}_$k.csv 2>/dev/null
  ncu -i $R --page source --csv > /tmp/src_$k.csv 2>/dev/null && python tools/ncu_src.py /tmp/src_$k.csv 0.005 > gpurun_out/src_${TAG}_$k.txt 2>&1
done
ls -la gpurun_out/*.ncu-rep
python - <<'PY'
import glob, os
reps = sorted(glob.glob("gpurun_out/prof_*.ncu-rep"), key=os.path.getsize)
for r in reps[1:]:   # keep the smallest report whole, drop the rest
    os.remove(r)
PY
