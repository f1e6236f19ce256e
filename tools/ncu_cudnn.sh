#!/bin/bash
# Profile torch SDPA's cuDNN backend at the c4 SP=8 attention shape (for structural comparison with
# our attention kernel; library code, not on any product path).  Pass 1 lists the launches; pass 2
# captures the cuDNN-generated SDPA kernel with --set full.
set -x
mkdir -p gpurun_out/cd
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cd/launches.csv \
    python tools/ncu_cudnn_sdpa.py > gpurun_out/cd/pass1.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:cudnn_generated" -s 1 -c 1 \
    -o gpurun_out/cd/cudnn_sdpa_c4sp8 -f python tools/ncu_cudnn_sdpa.py > gpurun_out/cd/ncu.log 2>&1
tail -3 gpurun_out/cd/ncu.log
