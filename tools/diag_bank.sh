O=gpurun_out/diag
mkdir -p $O
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__sass_inst_executed_op_shared_ld.sum,smsp__sass_inst_executed_op_shared_st.sum,smsp__sass_inst_executed_op_shared_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:fs1_stream_kernel -c 1 --csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/conf_c3.csv 2> $O/conf_c3.err
timeout 900 ncu --section SourceCounters --clock-control none --import-source on -k regex:fs1_stream_kernel -c 1 -o $O/src_c3 -f python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/src.log 2>&1
ncu -i $O/src_c3.ncu-rep --page source --csv --print-source cuda,sass > $O/source_c3.csv 2>&1
head -3 $O/source_c3.csv | cut -c1-3000 > $O/source_hdr.txt
gzip -9 -f $O/source_c3.csv; rm -f $O/src_c3.ncu-rep
