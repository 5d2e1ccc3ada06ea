#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/dbg_bisect.py _ra1 22 > gpurun_out/c5_bisect22.log 2>&1
timeout 900 python tools/dbg_bisect.py _ra1 24 > gpurun_out/c5_bisect24.log 2>&1
echo done
