#!/bin/bash
# ncu evidence for the FP8 mode: launch list of one bench step (L2 kept
# between launches, as in the graphed step) and one --set full capture of the
# 56x56 3x3 fp8 conv (second conv_tc launch of the step).
set -e
python tools/one_step.py --mode fp8 --dump gpurun_out/fp8_step.json > gpurun_out/fp8_one_step.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none --nvtx --nvtx-include "step/" --csv --log-file gpurun_out/r2_fp8_launches.csv \
    python tools/one_step.py --mode fp8 > gpurun_out/fp8_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" \
    -k regex:conv_tc_kernel -s 1 -c 2 -o gpurun_out/r2_fp8_conv \
    python tools/one_step.py --mode fp8 > gpurun_out/fp8_ncu2.log 2>&1
