#!/bin/bash
# CTA shape variants, second pass: A/B
mkdir -p gpurun_out
A="timeout 900 python tools/ab.py --class-work --reps 2"
$A --config c5 --libs base,_c1d,_c2w20,_c1g,_hwc --flags 1 >> gpurun_out/c10_ab.jsonl 2>>gpurun_out/c10_ab.err
$A --config c4 --libs base,_c1d,_c2w20,_c1g --flags 1 >> gpurun_out/c10_ab.jsonl 2>>gpurun_out/c10_ab.err
$A --config c2 --libs base,_c1b,_c1a --flags 1,3 >> gpurun_out/c10_ab.jsonl 2>>gpurun_out/c10_ab.err
echo done
