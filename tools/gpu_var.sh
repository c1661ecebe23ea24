for B in 1024 8192 32768; do for sb in 128 32; do PE_SMALL_BLOCK=$sb B=$B WARM=3 CFG=3 python tools/variant_bench.py variants/ondemand.so 2>&1 | tail -1 | sed "s/^/sb=$sb B=$B /"; done; done
for sb in 128 32; do PE_SMALL_BLOCK=$sb B=65536 WARM=1 CFG=4 python tools/variant_bench.py variants/ondemand.so 2>&1 | tail -1 | sed "s/^/sb=$sb cfg4 /"; done
for lb in 256 8192; do python bench.py --metric search --leaf-batch $lb --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('search lb=$lb', d['value'], d['episodes_per_s_full_budget'])"; done
