#!/bin/bash
mkdir -p gpurun_out
A="timeout 900 python tools/ab.py --class-work --reps 2"
$A --config c3 --libs base,_rhash,_rhash3,_r3 --flags 0,1 >> gpurun_out/ab15.jsonl 2>>gpurun_out/ab15.err
$A --config c4 --libs base,_rhash,_rhash3,_r3 --flags 1 >> gpurun_out/ab15.jsonl 2>>gpurun_out/ab15.err
$A --config c2 --libs base,_rhash,_rhash3 --flags 1,3 >> gpurun_out/ab15.jsonl 2>>gpurun_out/ab15.err
$A --config c5 --libs base,_rhash,_rhash3 --flags 1 >> gpurun_out/ab15.jsonl 2>>gpurun_out/ab15.err
