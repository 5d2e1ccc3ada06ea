#!/bin/bash
# run-ahead CTA kernels (no CTA barriers, double-buffered bitmaps) A/B; class G work items; parity of the new base
mkdir -p gpurun_out
A="timeout 600 python tools/ab.py --class-work --reps 2"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or edge or giant or hub or sweep" > gpurun_out/c3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c3_pytest.log
$A --config c4 --libs base,_ra1,_ra2 --flags 1 >> gpurun_out/c3_ab.jsonl 2>>gpurun_out/c3_ab.err
$A --config c5 --libs base,_ra1,_ra2 --flags 1 >> gpurun_out/c3_ab.jsonl 2>>gpurun_out/c3_ab.err
$A --config c4 --algo app --libs base --flags 1 >> gpurun_out/c3_ab.jsonl 2>>gpurun_out/c3_ab.err
$A --config c4 --ordering split --libs base,_ra1 --flags 1 >> gpurun_out/c3_ab.jsonl 2>>gpurun_out/c3_ab.err
$A --config c4 --ordering split --algo app --libs base --flags 1 >> gpurun_out/c3_ab.jsonl 2>>gpurun_out/c3_ab.err
$A --config c2 --libs base,_ra1 --flags 1,3 >> gpurun_out/c3_ab.jsonl 2>>gpurun_out/c3_ab.err
echo done
