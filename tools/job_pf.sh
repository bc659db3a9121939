#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pf_launches.csv python tools/time_profile.py > gpurun_out/pf_ncu.log 2>&1
