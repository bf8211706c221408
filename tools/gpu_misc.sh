#!/bin/bash
# ad-hoc round-2 probes: K3w per-phase timing (probe build) and K1 fp64 warps-per-CTA A/B
O=gpurun_out/misc; mkdir -p $O
FS1_LIB=$PWD/gpurun_var/lib_probe.so timeout 300 python tools/phase_sep.py > $O/phase_sep.txt 2>&1; cat $O/phase_sep.txt
for c in e1_2000 e1_8000 e2_2000 e2_8000; do
  for k in 0 62; do
    timeout 300 python bench.py --config $c --kernel $k --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_${c}_$k.json 2> $O/b_${c}_$k.err
    python -c "import json;d=json.loads(open('$O/b_${c}_$k.json').read().strip().splitlines()[-1]);print('$c $k', d['config']['kernel'], round(d['ms_per_step'],3))" || tail -3 $O/b_${c}_$k.err
  done
done
