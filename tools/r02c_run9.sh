#!/bin/bash
# CTA shape variants for C1 / H-wide: A/B
mkdir -p gpurun_out
A="timeout 900 python tools/ab.py --class-work --reps 2"
$A --config c5 --libs base,_c1a,_c1b,_c1c,_hwa --flags 1 >> gpurun_out/c9_ab.jsonl 2>>gpurun_out/c9_ab.err
$A --config c4 --libs base,_c1a,_c1b,_c1c --flags 1 >> gpurun_out/c9_ab.jsonl 2>>gpurun_out/c9_ab.err
echo done
