for l in base nolastdelta base nolastdelta; do WARM=4 B=262144 CFG=3 python tools/variant_bench.py variants/$l.so 2>&1 | tail -1; done
for l in base nolastdelta; do WARM=1 B=65536 CFG=4 python tools/variant_bench.py variants/$l.so 2>&1 | tail -1; done
