#!/bin/bash
# Round evidence: bench lines (all configs + oracle arm), smoke, ncu launch lists and one
# full capture per dominant kernel, exported to csv summaries (no .ncu-rep kept).
O=gpurun_out/${TAG:-final}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 300 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
for c in c1 c3 c4 c5 e1_8000 e2_8000; do
  timeout 400 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
# the multi-GPU launch path at N = 1 (torchrun, NCCL) and the sharded driver (gathered / fused exchange)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 5 --warmup 3 > $O/bench_c2_torchrun.json 2> $O/bench_c2_torchrun.err
for f in 0 1; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 \
    tools/shard_dist_demo.py 24 20 $f 2>&1 | grep world >> $O/shard_dist.txt
done
timeout 300 python tools/time_shard_graph.py 24 50 > $O/shard_graph_timing.txt 2>&1
for c in c2 c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch_$c.log 2>&1
done
for spec in "c2 fs1_persist_solve" "c3 fs1_stream_kernel" "c4 fs1_sep2dw"; do
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
