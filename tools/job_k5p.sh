#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"scan_place" -c 1 -o gpurun_out/k5p python tools/ncu_indexless.py > gpurun_out/k5p.log 2>&1
