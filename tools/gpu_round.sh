#!/bin/bash
# One GPU session: build check, GPU tests, bench lines per config, ncu launch lists and full captures.
set -x
O=gpurun_out/${TAG:-run}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
for c in c3 c4 c1 c5; do
  timeout 400 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for c in c2 c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fs1_stream -s 1 -c 1 -o $O/prof_c3 \
  python tools/prof_stream.py 20 > $O/ncu_full_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fs1_sep2d -s 1 -c 1 -o $O/prof_c4 \
  python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fs1_persist -s 1 -c 1 -o $O/prof_c2 \
  python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full_c2.log 2>&1
for p in c3 c4 c2; do
  if [ -f $O/prof_$p.ncu-rep ]; then
    ncu -i $O/prof_$p.ncu-rep --page raw --csv > $O/raw_$p.csv 2>&1
    ncu -i $O/prof_$p.ncu-rep --page details --csv > $O/details_$p.csv 2>&1
    ncu -i $O/prof_$p.ncu-rep --page source --csv --print-source cuda,sass > $O/source_$p.csv 2>&1
  fi
done
for p in c3 c4 c2; do
  [ -f $O/source_$p.csv ] && python tools/ncu_lines.py $O/source_$p.csv 60 > $O/lines_$p.txt 2>&1 && gzip -9 $O/source_$p.csv
done
rm -f $O/*.ncu-rep
du -sh $O
ls -la $O
