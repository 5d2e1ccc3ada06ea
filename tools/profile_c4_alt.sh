#!/bin/bash
# ncu captures of the class G kernel (and the slowest other class) on C4 under the
# orderings / algorithm the degree-order A+- headline does not exercise:
# split order A+- and degree order A++.   tools/profile_c4_alt.sh <tag>
TAG=${1:-r02c}
mkdir -p gpurun_out
run() {  # name ordering algo
  CMD="python bench.py --config c4 --ordering $2 --algo $3 --steps 1 --warmup 1 --no-cpu-baseline"
  $CMD > gpurun_out/plain_${TAG}_$1.json 2> gpurun_out/plain_${TAG}_$1.err || return 1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
      --log-file gpurun_out/launches_${TAG}_$1.csv $CMD > gpurun_out/ncu_launch_${TAG}_$1.log 2>&1
  for k in giant:k_list_giant reg:k_list_reg; do
    n=${k%%:*}; re=${k##*:}
    R=gpurun_out/prof_${TAG}_$1_$n
    ncu --set full --clock-control none --import-source on -k "regex:$re" -s 0 -c 1 -o $R $CMD > gpurun_out/ncu_full_${TAG}_$1_$n.log 2>&1
    [ -f $R.ncu-rep ] || continue
    ncu -i $R.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_$1_$n.csv 2>/dev/null
    ncu -i $R.ncu-rep --page source --csv > /tmp/src_$1_$n.csv 2>/dev/null && python tools/ncu_src.py /tmp/src_$1_$n.csv 0.004 > gpurun_out/src_${TAG}_$1_$n.txt 2>&1
    rm -f $R.ncu-rep
  done
}
run split_apm split apm
run degree_app degree app
echo "profile_c4_alt done"
