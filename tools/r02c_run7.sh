#!/bin/bash
# run-ahead CTA kernels (fixed), C2 at 768 threads: A/B
mkdir -p gpurun_out
A="timeout 900 python tools/ab.py --class-work --reps 2"
$A --config c5 --libs base,_ra1,_ra2,_ra3,_c2t768 --flags 1 >> gpurun_out/c7_ab.jsonl 2>>gpurun_out/c7_ab.err
$A --config c4 --libs base,_ra1,_ra2,_ra3,_c2t768 --flags 1 >> gpurun_out/c7_ab.jsonl 2>>gpurun_out/c7_ab.err
$A --config c2 --libs base,_ra1 --flags 1,3,7 >> gpurun_out/c7_ab.jsonl 2>>gpurun_out/c7_ab.err
echo done
