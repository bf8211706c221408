#!/bin/bash
# Round-2 first GPU cycle: full GPU suite, pipe micro-benchmark, bench lines, K2 phase probe.
O=gpurun_out/${TAG:-r02a}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench.cu -o /tmp/ubench && /tmp/ubench > $O/ubench.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x ${PYK:+-k "$PYK"} > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 300 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in ${CFGS:-c4}; do
  timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python tools/phase_stream.py > $O/phase_stream.txt 2>&1
