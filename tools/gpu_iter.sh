#!/bin/bash
# Iteration cycle: selected GPU tests, bench lines (repeats), K2 phase probe, ubench.
O=gpurun_out/${TAG:-iter}
mkdir -p $O
if [ -n "$UB" ]; then nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench.cu -o /tmp/ubench && /tmp/ubench > $O/ubench.txt 2>&1; fi
if [ -n "$PYK" ]; then timeout 1500 python -m pytest tests -m gpu -q -x -k "$PYK" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log; fi
for c in ${CFGS:-}; do
  for r in 1 ${REP:-}; do
    timeout 400 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline ${BARGS:-} > $O/bench_${c}_$r.json 2> $O/bench_${c}_$r.err
    python -c "import json;d=json.loads(open('$O/bench_${c}_$r.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$c', d['config']['kernel'], round(d['ms_per_step'],3), '%.4g'%d['value'], r['bound'], r.get('frac'), r.get('frac_nominal'), d['clocks'])" || tail -5 $O/bench_${c}_$r.err
  done
done
if [ -n "$PHASE" ]; then timeout 300 python tools/phase_stream.py > $O/phase_stream.txt 2>&1; cat $O/phase_stream.txt; fi
