#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/v5_check.py small > gpurun_out/v5_small.txt 2>&1; echo "rc=$?" >> gpurun_out/v5_small.txt
grep -q "ALL OK" gpurun_out/v5_small.txt || exit 0
timeout 300 python tools/v5_check.py > gpurun_out/v5_full.txt 2>&1; echo "rc=$?" >> gpurun_out/v5_full.txt
APAX_V5_PACE=0 timeout 300 python tools/v5_check.py > gpurun_out/v5_full_nopace.txt 2>&1
