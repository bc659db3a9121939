for cfg in "8 1" "8 4" "10 4" "12 4" "12 8" "16 8" "16 4"; do set -- $cfg
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-chunks $1 --e2e-taper $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('chunks $1 taper $2', round(e['value'],2), round(e['ms_per_step'],3), round(e['indexless_decode']['value'],2))"
done
