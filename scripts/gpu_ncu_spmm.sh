timeout 300 python scripts/spmm_one.py 286 > gpurun_out/spmm_one.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_seg" -s 1 -c 1 \
   -o gpurun_out/prof_spmm286 python scripts/spmm_one.py 286 > gpurun_out/ncu_spmm.log 2>&1; echo ncu=$?
