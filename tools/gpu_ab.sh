O=gpurun_out/ab1; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "persist or api or extra or c_abi or bench or dist or e1 or e2" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
for lib in main two w16; do
  for c in c2 c5; do
    if [ $lib = main ]; then L=""; else L="FS1_LIB=$PWD/gpurun_var/lib_$lib.so"; fi
    env $L timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_${lib}_$c.json 2> $O/b_${lib}_$c.err
    python -c "import json;d=json.loads(open('$O/b_${lib}_$c.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$lib $c', d['config']['kernel'], round(d['ms_per_step'],3), '%.4g'%d['value'], r.get('frac'), d['clocks']['sm_mhz'])" || tail -3 $O/b_${lib}_$c.err
  done
done
