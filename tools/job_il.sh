#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/time_indexless.py > gpurun_out/il_time.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/il_launches.csv python tools/ncu_indexless.py > gpurun_out/il_ncu.log 2>&1
