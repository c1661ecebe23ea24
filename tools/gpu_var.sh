export WARM=4
for cfg in 3; do for l in base ondemand base ondemand; do B=262144 CFG=$cfg python tools/variant_bench.py variants/$l.so 2>&1 | tail -1; done; done
for l in base ondemand; do B=65536 WARM=1 CFG=4 python tools/variant_bench.py variants/$l.so 2>&1 | tail -1; done
