#!/bin/bash
# every randomised parity hunt over the seeds in $SEEDS (default "1 2 3") -> gpurun_out/fuzz_all.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{
for s in ${SEEDS:-1 2 3}; do
echo "== seed $s"
timeout 900 python tools/fuzz_parity.py 1500 $(( 1000 * s + 11 ))
FUZZ_MAXBLK=120 timeout 900 python tools/fuzz_parity.py 400 $(( 1000 * s + 12 ))
timeout 900 python tools/fuzz_v5.py 800 $(( 1000 * s + 13 ))
timeout 900 python tools/fuzz_corrupt.py 800 $(( 1000 * s + 14 ))
timeout 900 python tools/fuzz_cast.py 800 $(( 1000 * s + 15 ))
timeout 900 python tools/fuzz_trace.py 600 $(( 1000 * s + 16 ))
timeout 900 python tools/fuzz_range.py 500 $(( 1000 * s + 17 ))
timeout 900 python tools/fuzz_extremes.py 600 $(( 1000 * s + 18 ))
FUZZ_CAST_EXTREME=1 timeout 900 python tools/fuzz_cast.py 400 $(( 1000 * s + 19 ))
timeout 900 python tools/fuzz_offsets.py 300 $(( 1000 * s + 20 ))
done
} > gpurun_out/fuzz_all.txt 2>&1
echo rc=$? >> gpurun_out/fuzz_all.txt
