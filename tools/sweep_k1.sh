run() { python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --no-e2e --kernel $3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['kernel'], round(d['ms_per_step'],3))" 2>/dev/null || echo "$1 $3 unsupported"; }
timeout 900 python -m pytest tests -m gpu -q -x -k "persist or nonfinite or smoke" 2>&1 | tail -1
run c2 5 31; run c5 3 32; run c5 3 34; run c5 3 32; run c5 3 34
