# A/B of variant builds with a correctness pass on the candidate: CAND=name PT="tests..." PK="-k expr"
O=gpurun_out/${TAG:-ab}; mkdir -p $O
FS1_LIB=$PWD/gpurun_var/lib_$CAND.so timeout 900 python -m pytest $PT -m gpu -q -x $PK > $O/pytest_$CAND.log 2>&1; echo "rc=$?" >> $O/pytest_$CAND.log; tail -3 $O/pytest_$CAND.log
bash tools/gpu_ab.sh
