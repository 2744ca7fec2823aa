# SpMM binding-unit evidence (round 2): L1 carveout probe, and the L2->L1 fill
# (xbar2l1tex) and L1/L2 throughput breakdowns of the access-stream ceiling,
# the lab SpMM and the product SpMM.  Run under gpurun.
mkdir -p gpurun_out
python scripts/dbg/dump_csr.py 2 /tmp/csr2.bin > /dev/null
LAB_CARVE=1 ./scripts/dbg/spmm_lab /tmp/csr2.bin > gpurun_out/lab_carve.txt 2>&1; echo carve=$?
M="gpu__time_duration.sum,breakdown:l1tex__throughput.avg.pct_of_peak_sustained_elapsed,breakdown:lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum.per_second,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active"
LAB_NCU=1 timeout 900 ncu --clock-control none --metrics $M --csv ./scripts/dbg/spmm_lab /tmp/csr2.bin > gpurun_out/ncu_fabric_lab.csv 2> gpurun_out/ncu_fabric_lab.err; echo ncu_lab=$?
B="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 900 ncu --clock-control none --metrics $M --csv -k regex:"k_spmm_fused" -s 40 -c 3 $B > gpurun_out/ncu_fabric_prod.csv 2> gpurun_out/ncu_fabric_prod.err; echo ncu_prod=$?
