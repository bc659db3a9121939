#!/bin/bash
cd $GRAFT_REPO_ROOT
APAX_V5_RANK=0 TIMES_VARIANT=times5 TIMES_FN=apax_debug_cta_times5 timeout 300 python tools/cta_times.py cfg2 > gpurun_out/v5_times.txt 2>&1
