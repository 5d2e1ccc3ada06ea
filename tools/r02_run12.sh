#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest12.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest12.log
A="timeout 900 python tools/ab.py --class-work --reps 3"
$A --config c5 --flags 0,1 --reps 2 >> gpurun_out/ab12.jsonl 2>>gpurun_out/ab12.err
$A --config c4 --flags 0,1 >> gpurun_out/ab12.jsonl 2>>gpurun_out/ab12.err
$A --config c3 --flags 0,1 >> gpurun_out/ab12.jsonl 2>>gpurun_out/ab12.err
$A --config c2 --flags 1,3,7 >> gpurun_out/ab12.jsonl 2>>gpurun_out/ab12.err
