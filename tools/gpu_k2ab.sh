O=gpurun_out/k2ab; mkdir -p $O
for r in 1 2; do for k in 10 11 12; do
 timeout 300 python bench.py --config c3 --kernel $k --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_${k}_$r.json 2> $O/b_${k}_$r.err
 python -c "import json;d=json.loads(open('$O/b_${k}_$r.json').read().strip().splitlines()[-1]);print($k, d['config']['kernel'], round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 $O/b_${k}_$r.err
done; done
