#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_v3_kernel -c 1 -o gpurun_out/src_dec python tools/ncu_indexless.py > gpurun_out/src_dec.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:encode_v3_kernel -c 1 -o gpurun_out/src_enc python tools/ncu_indexless.py > gpurun_out/src_enc.log 2>&1
