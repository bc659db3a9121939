#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_v3_kernel -s 2 -c 1 -o gpurun_out/decp python tools/ncu_decode.py > gpurun_out/decp.log 2>&1
