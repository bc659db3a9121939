cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"chain_kernel" -c 1 -o gpurun_out/j15_wsfq python tools/time_encode.py "cfg2/16" > gpurun_out/j15_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"chain_kernel" -c 1 -o gpurun_out/j15_wsfr python tools/time_encode.py "cfg1 FR whole" >> gpurun_out/j15_ncu.log 2>&1
