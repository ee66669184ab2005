# Final round-2 profiles: launch list + K1 --set full (generation order), and the
# unordered-input path with the one-pass scatter (launch metrics + KQ1/KP2 --set full).
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu --quick"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02c.csv $B > gpurun_out/ncu_launch_c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_contract -c 1 -o gpurun_out/k1_r02c $B > gpurun_out/ncu_k1c.log 2>&1
S="python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu --order shuffled --quick"
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum -k regex:"k_part|k_compact|k_bkt|k_sorted|k_col|k_table_clear|k_order" -c 40 --csv --log-file gpurun_out/shuf_r02c_metrics.csv $S > gpurun_out/ncu_shuf_c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_part_stream|k_part_agg" -c 2 -o gpurun_out/kq_r02c $S > gpurun_out/ncu_kq_c.log 2>&1
echo profiles done
