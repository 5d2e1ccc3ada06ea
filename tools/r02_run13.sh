#!/bin/bash
mkdir -p gpurun_out
A="timeout 900 python tools/ab.py --class-work --reps 2"
$A --config c4 --ordering split --libs base,_g24,_g48,_g74 --flags 1 >> gpurun_out/ab13.jsonl 2>>gpurun_out/ab13.err
$A --config c4 --algo app --libs base,_g24,_g48,_g74 --flags 1 >> gpurun_out/ab13.jsonl 2>>gpurun_out/ab13.err
