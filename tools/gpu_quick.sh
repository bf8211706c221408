#!/bin/bash
# Quick GPU cycle: selected GPU tests + bench lines.  usage: TAG=x bash tools/gpu_quick.sh "<pytest -k expr>" "<configs>"
O=gpurun_out/${TAG:-quick}
mkdir -p $O
K="${1:-}"
timeout 900 python -m pytest tests -m gpu -q -x ${K:+-k "$K"} > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for c in ${2:-}; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json;d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1]);print('$c', d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'), d['config'].get('kernel'))" || tail -5 $O/bench_$c.err
done
