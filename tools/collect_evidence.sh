#!/bin/bash
# Copy one gpu_final.sh evidence set (gpurun_out/$TAG) into profiles/r02/${TAG}_* and
# refresh profiles/traffic.json from its full captures.
T=${1:?tag}; S=gpurun_out/$T; D=profiles/r02
for f in $S/bench_*.json; do cp $f $D/${T}_$(basename $f); done
for f in $S/launches_*.csv; do cp $f $D/${T}_$(basename $f); done
for f in $S/summary_*.txt; do b=$(basename $f .txt); cp $f $D/${T}_ncu_${b#summary_}.txt; done
for f in $S/lines_*.txt; do b=$(basename $f .txt); cp $f $D/${T}_srclines_${b#lines_}.txt; done
tail -5 $S/pytest_gpu.log > $D/${T}_pytest_gpu_tail.txt
cp $S/smoke.log $D/${T}_smoke.log; cp $S/smi.txt $D/${T}_smi.txt
cp $S/golden_errors.txt $D/golden_errors.txt
python - "$T" <<'PY'
import json, sys, glob, os
T = sys.argv[1]
p = "profiles/traffic.json"; d = json.load(open(p))
for f in glob.glob(f"profiles/r02/{T}_ncu_*.txt"):
    cfg = os.path.basename(f)[len(T) + 5:-4]
    rd = wr = None
    for line in open(f):
        k = line.split()
        if not k: continue
        if k[0] == "dram__bytes_read.sum": rd = float(k[1]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[k[2]] if len(k) > 2 else float(k[1])
        if k[0] == "dram__bytes_write.sum": wr = float(k[1]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[k[2]] if len(k) > 2 else float(k[1])
    if rd is not None and wr is not None: d[cfg] = int(rd + wr)
d["_note"] = d["_note"].split(" (profiles/")[0] + f" (profiles/r02/{T}_ncu_*.txt where captured, else the earlier sets)"
json.dump(d, open(p, "w"), indent=1)
print(d)
PY
