#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:encode_v5_kernel -s 2 -c 1 -o gpurun_out/v5p python tools/ncu_enc.py 0 > gpurun_out/v5p.log 2>&1
