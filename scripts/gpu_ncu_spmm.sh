# ncu --set full of the SpMM launches of the third 286-column and 128-column application (configs[2])
for spec in "286 8 4" "128 4 2"; do
set -- $spec
timeout 300 python scripts/spmm_one.py $1 > gpurun_out/spmm_one_$1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm" -s $2 -c $3 \
   -o gpurun_out/prof_spmm$1 python scripts/spmm_one.py $1 > gpurun_out/ncu_spmm$1.log 2>&1; echo ncu$1=$?
done
