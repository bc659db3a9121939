#!/bin/bash
# randomised parity hunt (tools/fuzz_parity.py, fuzz_v5.py, fuzz_corrupt.py) with fresh seeds
cd /root/repo
mkdir -p gpurun_out
{
echo "== fuzz_parity small"; timeout 500 python tools/fuzz_parity.py 500 ${SEED:-4242}
echo "== fuzz_parity long"; FUZZ_MAXBLK=90 timeout 700 python tools/fuzz_parity.py 250 $(( ${SEED:-4242} + 1 ))
echo "== fuzz_v5"; timeout 600 python tools/fuzz_v5.py 300 $(( ${SEED:-4242} + 2 ))
echo "== fuzz_corrupt"; timeout 600 python tools/fuzz_corrupt.py 300 $(( ${SEED:-4242} + 3 ))
} > gpurun_out/fuzz.txt 2>&1
echo rc=$? >> gpurun_out/fuzz.txt
