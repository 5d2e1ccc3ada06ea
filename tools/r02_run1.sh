#!/bin/bash
# round-2 check 1: GPU suite after the ADVICE fixes, per-class A/B on C4, new bench arms on C4
mkdir -p gpurun_out
df -h /dev/shm /tmp > gpurun_out/df.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
for f in 0 1; do timeout 300 python tools/ab.py --config c4 --flags $f >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err; done
TRIGPU_LIB_SUFFIX=_exp timeout 300 python tools/ab.py --config c4 --flags 0 --variant 2 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?" >> gpurun_out/bench_c4.err
timeout 900 python bench.py --impl reference --config c4 --steps 2 --warmup 1 > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err; echo "ref rc=$?" >> gpurun_out/ref_c4.err
