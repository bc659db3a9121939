#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/v5_check.py small > gpurun_out/v5_small.txt 2>&1; echo "rc=$?" >> gpurun_out/v5_small.txt
grep -q "ALL OK" gpurun_out/v5_small.txt || exit 0
timeout 300 python tools/v5_check.py > gpurun_out/v5_full.txt 2>&1; echo "rc=$?" >> gpurun_out/v5_full.txt
timeout 300 python tools/prof_v5.py > gpurun_out/v5_prof.txt 2>&1
