# Final build, unordered-input path (config 4 in a seeded random order): launch metrics of one step
cd $GRAFT_REPO_ROOT
S="python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu --order shuffled --quick"
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum -k regex:"k_part|k_compact|k_bkt|k_sorted|k_col|k_table_clear|k_order|k_find" -c 40 --csv --log-file gpurun_out/shuf_r02d_metrics.csv $S > gpurun_out/ncu_shuf_d.log 2>&1
echo done
