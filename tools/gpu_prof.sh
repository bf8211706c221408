#!/bin/bash
# One full ncu capture of kernel regex $2 in `python bench.py --config $1`, exported to csv summaries.
# usage: TAG=x bash tools/gpu_prof.sh c4 fs1_sep2dw [extra bench args]
O=gpurun_out/${TAG:-prof}
mkdir -p $O
C=$1; K=$2; shift 2
CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $*"
timeout 300 $CMD > $O/plain_$C.log 2>&1 || { echo "plain run failed"; tail -5 $O/plain_$C.log; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $O/prof_$C -f $CMD > $O/ncu_$C.log 2>&1
ncu -i $O/prof_$C.ncu-rep --page raw --csv > $O/raw_$C.csv 2>&1
ncu -i $O/prof_$C.ncu-rep --page source --csv --print-source cuda,sass > $O/source_$C.csv 2>&1
python tools/ncu_summary.py $O/raw_$C.csv > $O/summary_$C.txt 2>&1
python tools/ncu_lines.py $O/source_$C.csv 50 > $O/lines_$C.txt 2>&1
gzip -9 -f $O/source_$C.csv
rm -f $O/prof_$C.ncu-rep
cat $O/summary_$C.txt; head -30 $O/lines_$C.txt
