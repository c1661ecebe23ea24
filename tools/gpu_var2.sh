# code-size variants (tools/build_variants.sh): config 3 at the bench step, config 4 at 64K
mkdir -p gpurun_out
for r in 1 2; do for v in base le legd; do WARM=2 B=1048576 CFG=3 timeout 300 python tools/variant_bench.py variants/$v.so 2>&1 | tail -1 | sed "s/^/cfg3 r$r /"; done; done
for v in base le legd; do WARM=1 B=65536 CFG=4 timeout 600 python tools/variant_bench.py variants/$v.so 2>&1 | tail -1 | sed "s/^/cfg4 /"; done
