#!/bin/bash
# randomised parity hunt (tools/fuzz_parity.py, fuzz_v5.py, fuzz_corrupt.py) over several seeds
cd /root/repo
mkdir -p gpurun_out
{
for s in ${SEEDS:-1 2 3}; do
echo "== seed $s fuzz_parity small"; timeout 900 python tools/fuzz_parity.py 1500 $(( 1000 * s + 11 ))
echo "== seed $s fuzz_parity long"; FUZZ_MAXBLK=120 timeout 900 python tools/fuzz_parity.py 400 $(( 1000 * s + 12 ))
echo "== seed $s fuzz_v5"; timeout 900 python tools/fuzz_v5.py 800 $(( 1000 * s + 13 ))
echo "== seed $s fuzz_corrupt"; timeout 900 python tools/fuzz_corrupt.py 800 $(( 1000 * s + 14 ))
done
} > gpurun_out/fuzz.txt 2>&1
echo rc=$? >> gpurun_out/fuzz.txt
