# ncu evidence for the unordered-input path with the one-pass scatter (config 4, seeded random order)
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu --order shuffled --quick"
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum -k regex:"k_part|k_compact|k_bkt|k_sorted|k_col|k_table_clear|k_order" -c 40 --csv --log-file gpurun_out/shuf2_metrics.csv $B > gpurun_out/ncu_shuf2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_part_stream|k_part_agg" -c 2 -o gpurun_out/kq_full $B > gpurun_out/ncu_kq.log 2>&1
