for B in 4096 8192 16384 32768 65536 131072; do for c in 32 0; do PE_CPW=$c WARM=3 B=$B CFG=3 python tools/variant_bench.py variants/solo.so 2>&1 | tail -1 | sed "s/^/cfg3 cpw=$c B=$B /"; done; done
for B in 4096 16384 65536; do for c in 32 0; do PE_CPW=$c WARM=1 B=$B CFG=4 python tools/variant_bench.py variants/solo.so 2>&1 | tail -1 | sed "s/^/cfg4 cpw=$c B=$B /"; done; done
