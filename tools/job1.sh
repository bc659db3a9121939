cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/j1_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/j1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/j1_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/j1_bench.json 2> gpurun_out/j1_bench.err; echo "bench rc=$?" >> gpurun_out/j1_bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/j1_ref.json 2> gpurun_out/j1_ref.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"encode_v3" -s 3 -c 1 -o gpurun_out/j1_enc python bench.py --steps 2 --warmup 3 --profile > gpurun_out/j1_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/j1_ncu.log
