run() { python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --kernel $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['kernel'], d['config']['iters'], round(d['ms_per_step'],3))" 2>/dev/null || echo "$1 $2 unsupported"; }
for k in 0 32 34 38; do run c1 $k; done
