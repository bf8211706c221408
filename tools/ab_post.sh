# K2s (shard) GPU tests on the main build, the 2D tests on the AGGNF candidate, C4 A/B, shard timing
O=gpurun_out/ab4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_sep2d.py -m gpu -q -x > $O/pytest_main.log 2>&1; echo "rc=$?" >> $O/pytest_main.log; tail -3 $O/pytest_main.log
FS1_LIB=$PWD/gpurun_var/lib_nf.so timeout 900 python -m pytest tests/test_gpu_sep2d.py tests/test_gpu_golden.py -m gpu -q -x -k "sep2d or c4" > $O/pytest_nf.log 2>&1; echo "rc=$?" >> $O/pytest_nf.log; tail -3 $O/pytest_nf.log
timeout 600 python tools/time_shard_graph.py > $O/time_shard_graph.txt 2>&1; tail -5 $O/time_shard_graph.txt
TAG=ab4 REP=2 LIBS="main nf" CFGS=c4 bash tools/gpu_ab.sh
