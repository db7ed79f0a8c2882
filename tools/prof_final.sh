#!/bin/bash
# Round-2 final ncu evidence (run under gpurun after the plain commands exited 0):
#  * launch list of one bf16 ResNet-50 b64 bench step (the recipe's
#    gpu__time_duration pass; cold cache, serialised)
#  * launch list of one Inception-v3 b128 step (after the geometry rule)
#  * one --set full capture of a 28x28 3x3 conv and a 56x56 residual 1x1
set -e
python tools/one_step.py --dump gpurun_out/r2f_step.json > gpurun_out/r2f_one_step.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --nvtx --nvtx-include "step/" --csv --log-file gpurun_out/r2f_launches.csv \
    python tools/one_step.py > gpurun_out/r2f_ncu1.log 2>&1
python tools/one_step.py --model inception_v3 --batch 128 --dump gpurun_out/r2f_inc_step.json > gpurun_out/r2f_inc_one_step.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --nvtx --nvtx-include "step/" --csv --log-file gpurun_out/r2f_inc_launches.csv \
    python tools/one_step.py --model inception_v3 --batch 128 > gpurun_out/r2f_inc_ncu1.log 2>&1
# conv_tc launches of the ResNet step in order: conv11, conv19, conv34, conv27, ... conv101 is the 12th
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" \
    -k regex:conv_tc_kernel -s 3 -c 1 -o gpurun_out/r2f_conv27 \
    python tools/one_step.py > gpurun_out/r2f_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" \
    -k regex:conv_tc_kernel -s 11 -c 1 -o gpurun_out/r2f_conv101 \
    python tools/one_step.py > gpurun_out/r2f_ncu3.log 2>&1
