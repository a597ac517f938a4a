# per-kernel launch list of the hierarchical benchmark (2048^3): time and DRAM bytes
mkdir -p gpurun_out/hp
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_seed|k_upsample|k_gather|k_contract|k_fill|k_pyramid|k_resident" --csv --log-file gpurun_out/hp/l.csv python tools/bench_hier.py --scale ${SCALE:-1.0} > gpurun_out/hp/o.log 2>&1; echo rc=$?
