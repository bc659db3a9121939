#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/il_launches.csv python tools/ncu_indexless.py > gpurun_out/il_ncu.log 2>&1
