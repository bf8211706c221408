#!/bin/bash
# A/B of variant libraries on one config: usage TAG=x bash tools/ab_var.sh <config> "<pytest -k expr>" var1 var2 ...
# ("main" = the in-tree libfs1.so, else gpurun_var/lib_<var>.so via FS1_LIB); the tests run on the FIRST variant.
O=gpurun_out/${TAG:-ab}; mkdir -p $O
C=$1; K=$2; shift 2
if [ -n "$K" ]; then
  if [ $1 != main ]; then export FS1_LIB=$PWD/gpurun_var/lib_$1.so; fi
  timeout 900 python -m pytest tests -m gpu -q -x -k "$K" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
  tail -3 $O/pytest.log; unset FS1_LIB
fi
for i in 1 2 3; do
  for v in "$@"; do
    if [ $v = main ]; then unset FS1_LIB; else export FS1_LIB=$PWD/gpurun_var/lib_$v.so; fi
    timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${C}_${v}_$i.json 2> $O/bench_${C}_${v}_$i.err
    python -c "import json;d=json.loads(open('$O/bench_${C}_${v}_$i.json').read().strip().splitlines()[-1]);print('$v', d['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
