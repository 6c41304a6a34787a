#!/bin/bash
mkdir -p gpurun_out/r02p
RB_SWEEP_DELAY=16 ROWBLOCK_B200_LIB=variants/noload.so timeout 300 python tools/spmm_once.py 5 1 2 > gpurun_out/r02p/noload.log 2>&1
RB_SWEEP_DELAY=16 ROWBLOCK_B200_LIB=variants/prof.so timeout 300 python tools/spmm_once.py 5 1 2 > gpurun_out/r02p/prof_d16.log 2>&1
