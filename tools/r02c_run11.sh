#!/bin/bash
# exact per-warp hash probe for class R (TRIGPU_R_HASH) vs the windowed bitmap: A/B; C2 with the class-H split
mkdir -p gpurun_out
A="timeout 900 python tools/ab.py --class-work --reps 3"
$A --config c3 --libs base,_rhash --flags 0,1,3 >> gpurun_out/c13_ab.jsonl 2>>gpurun_out/c13_ab.err
$A --config c2 --libs base,_rhash --flags 1,3,7 >> gpurun_out/c13_ab.jsonl 2>>gpurun_out/c13_ab.err
$A --config c4 --libs base,_rhash --flags 1 >> gpurun_out/c13_ab.jsonl 2>>gpurun_out/c13_ab.err
$A --config c5 --libs base,_rhash --flags 1 >> gpurun_out/c13_ab.jsonl 2>>gpurun_out/c13_ab.err
echo done
