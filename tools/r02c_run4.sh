#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/dbg_lib.py _ra1 18 > gpurun_out/c4_dbg_plain.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/dbg_lib.py _ra1 16 > gpurun_out/c4_dbg_memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/dbg_lib.py _ra1 15 > gpurun_out/c4_dbg_racecheck.log 2>&1
echo done
