#!/bin/bash
# last validation of the round on the committed kernels: both GPU suites, C5 / C4 bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/f3_pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f3_pytest_parity.log
timeout 900 python bench.py > gpurun_out/f3_bench_c5.json 2> gpurun_out/f3_bench_c5.err; echo "rc=$?" >> gpurun_out/f3_bench_c5.err
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/f3_bench_c4.json 2> gpurun_out/f3_bench_c4.err
timeout 900 python tools/ab.py --class-work --reps 2 --config c5 --libs base,_c1d512 --flags 1 >> gpurun_out/f3_ab.jsonl 2>>gpurun_out/f3_ab.err
timeout 900 python tools/ab.py --class-work --reps 2 --config c4 --libs base,_c1d512 --flags 1 >> gpurun_out/f3_ab.jsonl 2>>gpurun_out/f3_ab.err
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/f3_pytest_fullsize.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f3_pytest_fullsize.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1
echo done
