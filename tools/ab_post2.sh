# 2D tests + C4 golden on the main build (K3w AGGNF on), the test on the pre-change build, C3 A/B of the scan variant
O=gpurun_out/ab5; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sep2d.py tests/test_gpu_golden.py tests/test_gpu_paper_e3.py -m gpu -q > $O/pytest_main.log 2>&1; echo "rc=$?" >> $O/pytest_main.log; tail -3 $O/pytest_main.log
FS1_LIB=$PWD/gpurun_var/lib_pf.so timeout 300 python -m pytest tests/test_gpu_sep2d.py -m gpu -q -k nonfinite > $O/pytest_old.log 2>&1; echo "rc=$?" >> $O/pytest_old.log; tail -2 $O/pytest_old.log
FS1_LIB=$PWD/gpurun_var/lib_sm.so timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_persist.py -m gpu -q -x > $O/pytest_sm.log 2>&1; echo "rc=$?" >> $O/pytest_sm.log; tail -2 $O/pytest_sm.log
TAG=ab5 REP=2 LIBS="main sm" CFGS="c3 c2" bash tools/gpu_ab.sh
