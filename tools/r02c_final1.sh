#!/bin/bash
# round 2 (session 4) validation: both GPU suites, the C5 bench line, the reference arm, C4, the C5 launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/f1_smi.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/f1_pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f1_pytest_parity.log
timeout 900 python bench.py > gpurun_out/f1_bench_c5.json 2> gpurun_out/f1_bench_c5.err; echo "rc=$?" >> gpurun_out/f1_bench_c5.err
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/f1_bench_c4.json 2> gpurun_out/f1_bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/f1_launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/f1_ncu.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/f1_pytest_fullsize.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f1_pytest_fullsize.log
echo done
