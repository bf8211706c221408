#!/bin/bash
# one ncu --set full capture of the dominant kernel of one config: CFG=e2s_8000 KRE=fs1_stab
O=gpurun_out/${TAG:-prof1}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 1 -c 1 -o $O/prof -f \
  python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
ncu -i $O/prof.ncu-rep --page raw --csv > $O/raw.csv 2>&1
ncu -i $O/prof.ncu-rep --page source --csv --print-source cuda,sass > $O/source.csv 2>&1
python tools/ncu_summary.py $O/raw.csv > $O/summary.txt 2>&1
python tools/ncu_lines.py $O/source.csv 40 > $O/lines.txt 2>&1
rm -f $O/prof.ncu-rep $O/source.csv
head -20 $O/summary.txt; head -30 $O/lines.txt
