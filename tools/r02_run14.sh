#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest14.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest14.log
A="timeout 900 python tools/ab.py --class-work --reps 2"
$A --config c4 --ordering split --flags 1 >> gpurun_out/ab14.jsonl 2>>gpurun_out/ab14.err
$A --config c4 --algo app --flags 1 >> gpurun_out/ab14.jsonl 2>>gpurun_out/ab14.err
$A --config c2 --flags 0,3,7 >> gpurun_out/ab14.jsonl 2>>gpurun_out/ab14.err
$A --config c2 --ordering split --algo app --flags 1 >> gpurun_out/ab14.jsonl 2>>gpurun_out/ab14.err
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c2_list or c3_1m" > gpurun_out/pytest14b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest14b.log
