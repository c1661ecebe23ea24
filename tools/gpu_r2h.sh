for d in bis_269a37b . bis_269a37b .; do
(cd $d && python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-parity-sample 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', d['value'], d['ms_per_step'])")
done
