#!/bin/bash
# final validation of the round: parity suite, C5 / C4 bench lines, C5 launch list,
# ncu --set full of the C5 class-H (warp + CTA) and C1 kernels, C4 split / A++ captures
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/f2_pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f2_pytest_parity.log
timeout 900 python bench.py > gpurun_out/f2_bench_c5.json 2> gpurun_out/f2_bench_c5.err; echo "rc=$?" >> gpurun_out/f2_bench_c5.err
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/f2_bench_c4.json 2> gpurun_out/f2_bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/f2_launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/f2_ncu.log 2>&1
TAG=r02d
CMD="python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline"
prof() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 \
      -o gpurun_out/prof_${TAG}_$1 $CMD > gpurun_out/ncu_full_${TAG}_$1.log 2>&1
  R=gpurun_out/prof_${TAG}_$1.ncu-rep
  [ -f "$R" ] || return
  ncu -i $R --page raw --csv > gpurun_out/raw_${TAG}_$1.csv 2>/dev/null
  ncu -i $R --page source --csv > /tmp/src_$1.csv 2>/dev/null && python tools/ncu_src.py /tmp/src_$1.csv 0.004 > gpurun_out/src_${TAG}_$1.txt 2>&1
  rm -f $R
}
prof warp_h k_list_warp 0
prof cta_h k_list_cta 0
prof cta_c1 k_list_cta 1
bash tools/profile_c4_alt.sh r02d
echo done
