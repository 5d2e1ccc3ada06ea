#!/bin/bash
# occupancy variants (C1 / H-wide at 4 CTAs per SM) and the lane-per-row path of class R: A/B
mkdir -p gpurun_out
A="timeout 900 python tools/ab.py --class-work --reps 2"
timeout 300 python tools/dbg_lib.py _lr 18 > gpurun_out/c8_dbg_lr.log 2>&1
$A --config c3 --libs base,_lr --flags 0,1,3 >> gpurun_out/c8_ab.jsonl 2>>gpurun_out/c8_ab.err
$A --config c5 --libs base,_c1m4,_hw18m4,_lr --flags 1 >> gpurun_out/c8_ab.jsonl 2>>gpurun_out/c8_ab.err
$A --config c4 --libs base,_c1m4,_lr --flags 1 >> gpurun_out/c8_ab.jsonl 2>>gpurun_out/c8_ab.err
$A --config c2 --libs base,_c1m4,_lr --flags 1,3,7 >> gpurun_out/c8_ab.jsonl 2>>gpurun_out/c8_ab.err
echo done
