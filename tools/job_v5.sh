#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/v5_check.py small > gpurun_out/v5_small.txt 2>&1; echo "rc=$?" >> gpurun_out/v5_small.txt
