#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest11.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest11.log
timeout 1200 python tools/ab.py --config c5 --libs base,_c1w19,_c2w20,_rw16,_hc19 --flags 1 --reps 2 --class-work >> gpurun_out/ab11.jsonl 2>>gpurun_out/ab11.err
timeout 600 python tools/ab.py --config c4 --libs base --flags 1 --reps 2 >> gpurun_out/ab11.jsonl 2>>gpurun_out/ab11.err
timeout 600 python tools/ab.py --config c3 --libs base --flags 1 --reps 2 >> gpurun_out/ab11.jsonl 2>>gpurun_out/ab11.err
