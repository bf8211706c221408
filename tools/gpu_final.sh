#!/bin/bash
# Round evidence: full GPU suite, bench lines for every config and the oracle arm, smoke,
# ncu launch lists and one full capture per dominant kernel (csv summaries; no .ncu-rep kept).
O=gpurun_out/${TAG:-final}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
if [ -z "$NOTEST" ]; then
  timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  tail -3 $O/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python tools/golden_errors.py > $O/golden_errors.txt 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in ${CFGS:-c1 c2 c4 c5 e1_8000 e2_8000 e2s_8000 e3_160 e3_80}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 5 --warmup 3 > $O/bench_c3_torchrun.json 2> $O/bench_c3_torchrun.err
for c in ${LCFGS:-c3 c2 c4 c5}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch_$c.log 2>&1
done
# PCFGS: comma-separated "config kernel-regex" pairs
IFS=, read -ra SPECS <<< "${PCFGS:-c3 fs1_stream_kernel,c4 fs1_sep2dw,c5 fs1_persist_solve,c2 fs1_persist_solve,e3_160 fs1_sep2d64w,e2s_8000 fs1_stab}"
for spec in "${SPECS[@]}"; do
  set -- $spec
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o $O/prof_$1 -f \
    python bench.py --config $1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full_$1.log 2>&1
  ncu -i $O/prof_$1.ncu-rep --page raw --csv > $O/raw_$1.csv 2>&1
  ncu -i $O/prof_$1.ncu-rep --page source --csv --print-source cuda,sass > $O/source_$1.csv 2>&1
  python tools/ncu_summary.py $O/raw_$1.csv > $O/summary_$1.txt 2>&1
  python tools/ncu_lines.py $O/source_$1.csv 40 > $O/lines_$1.txt 2>&1
  gzip -9 -f $O/source_$1.csv
  rm -f $O/prof_$1.ncu-rep
done
du -sh $O
