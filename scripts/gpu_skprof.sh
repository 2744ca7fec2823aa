timeout 300 python scripts/sketch_one.py > gpurun_out/sketch_one.log 2>&1; echo one=$?
tail -3 gpurun_out/sketch_one.log
timeout 300 python scripts/sketch_one.py > gpurun_out/sketch_one2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sketch_tc" -s 2 -c 2 \
   -o gpurun_out/prof_sketch python scripts/sketch_one.py > gpurun_out/ncu_sketch.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_sketch.log
