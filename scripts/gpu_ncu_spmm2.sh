for v in 9 21; do
NETMFP_SPMM=$v timeout 300 python scripts/spmm_one.py 128 > gpurun_out/spmm_one_$v.log 2>&1 && \
NETMFP_SPMM=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_rows|k_spmm_wr" -s 1 -c 1 \
   -o gpurun_out/prof_spmm_v$v python scripts/spmm_one.py 128 > gpurun_out/ncu_spmm_$v.log 2>&1; echo ncu$v=$?
done
