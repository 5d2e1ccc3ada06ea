#!/bin/bash
mkdir -p gpurun_out
A="timeout 900 python tools/ab.py --class-work --reps 2"
$A --config c5 --flags 0,1 >> gpurun_out/ab9.jsonl 2>>gpurun_out/ab9.err
$A --config c4 --flags 1 >> gpurun_out/ab9.jsonl 2>>gpurun_out/ab9.err
$A --config c4 --ordering split --flags 1 >> gpurun_out/ab9.jsonl 2>>gpurun_out/ab9.err
$A --config c4 --algo app --flags 1 >> gpurun_out/ab9.jsonl 2>>gpurun_out/ab9.err
$A --config c3 --flags 1 >> gpurun_out/ab9.jsonl 2>>gpurun_out/ab9.err
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest9.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest9.log
