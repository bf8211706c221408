#!/bin/bash
# A/B timing of variant builds (tools/variant.sh): LIBS="main x y" CFGS="c4" PYK="pytest -k expr"
O=gpurun_out/${TAG:-ab}; mkdir -p $O
if [ -n "$PYK" ]; then timeout 1200 python -m pytest tests -m gpu -q -x -k "$PYK" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log; fi
for r in 1 ${REP:-}; do
for lib in ${LIBS:-main}; do
  for c in ${CFGS:-c4}; do
    if [ $lib = main ]; then L=""; else L="FS1_LIB=$PWD/gpurun_var/lib_$lib.so"; fi
    env $L timeout 300 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e ${BARGS:-} > $O/b_${lib}_${c}_$r.json 2> $O/b_${lib}_${c}_$r.err
    python -c "import json;d=json.loads(open('$O/b_${lib}_${c}_$r.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$lib $c', d['config']['kernel'], round(d['ms_per_step'],3), '%.4g'%d['value'], r.get('frac'), d['clocks']['sm_mhz'])" || tail -3 $O/b_${lib}_${c}_$r.err
  done
done
done
