#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python tools/ncu_enc.py > gpurun_out/s4b_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:encode_v3_kernel -s 2 -c 1 -o gpurun_out/s4b_fused python tools/ncu_enc.py 0 > gpurun_out/s4b_fused.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"encode_v3_kernel|pack_kernel" -s 4 -c 2 -o gpurun_out/s4b_split python tools/ncu_enc.py 1 > gpurun_out/s4b_split.log 2>&1
