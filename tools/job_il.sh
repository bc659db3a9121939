#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_place_kernel -s 3 -c 1 -o gpurun_out/scanp python tools/ncu_indexless.py > gpurun_out/scanp.log 2>&1
