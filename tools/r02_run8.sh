#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/ab.py --config c4 --libs base,_lea,_h15,_h15m4,_c1m4,_h15c1m4 --flags 0,1 >> gpurun_out/ab8.jsonl 2>>gpurun_out/ab8.err
timeout 900 python tools/ab.py --config c5 --libs base,_lea,_h15,_c1m4,_h15c1m4 --flags 1 --reps 2 >> gpurun_out/ab8.jsonl 2>>gpurun_out/ab8.err
