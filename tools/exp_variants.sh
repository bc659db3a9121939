#!/bin/bash
# bench.py device-only legs for each (variant, P): tools/exp_variants.sh "v1 v2" "28 37"
cd "$(dirname "$0")/.."
for v in $1; do
  for p in $2; do
    if [ "$v" = "product" ]; then lib=""; else lib="APAX_LIB_PATH=$PWD/build_variants/$v/libapax_b200.so"; fi
    r=$(env $lib timeout 300 python bench.py --workload ${WL:-cfg2} --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --segment-blocks $p 2>&1 | tail -1)
    echo "$v P=$p $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("enc %.4f dec %.4f ratio %.4f value %.1f" % (d["encode_ms"], d["decode_ms"], d["ratio"], d["value"]))' 2>&1)"
  done
done
