#!/bin/bash
# validate: vcount sink, class G window, R queue batching, single-pass list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest6.log
A="timeout 600 python tools/ab.py --reps 3"
$A --config c4 --flags 0,1 >> gpurun_out/ab6.jsonl 2>>gpurun_out/ab6.err
$A --config c4 --ordering split --flags 1 >> gpurun_out/ab6.jsonl 2>>gpurun_out/ab6.err
$A --config c4 --algo app --flags 1 >> gpurun_out/ab6.jsonl 2>>gpurun_out/ab6.err
$A --config c2 --flags 3,7 >> gpurun_out/ab6.jsonl 2>>gpurun_out/ab6.err
$A --config c3 --flags 1 >> gpurun_out/ab6.jsonl 2>>gpurun_out/ab6.err
$A --config c2 --ordering split --algo app --flags 1 --reps 2 >> gpurun_out/ab6.jsonl 2>>gpurun_out/ab6.err
