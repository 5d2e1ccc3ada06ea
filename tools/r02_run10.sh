#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/ab.py --config c5 --libs base,_hc18m3,_hc17m4,_hc19m3 --flags 1 --reps 2 --class-work >> gpurun_out/ab10.jsonl 2>>gpurun_out/ab10.err
timeout 900 python tools/ab.py --config c4 --libs base,_hc18m3,_hc17m4,_hc19m3 --flags 0,1 --reps 3 --class-work >> gpurun_out/ab10.jsonl 2>>gpurun_out/ab10.err
