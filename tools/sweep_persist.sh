run() { python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --no-e2e --kernel $3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['kernel'], round(d['ms_per_step'],3))" 2>/dev/null || echo "$1 $3 unsupported"; }
for k in 31 32 34 38; do run c2 5 $k; done
for k in 32 34 38 46; do run c5 3 $k; done
for k in 34 38 46; do run c1 5 $k; done
