set -x
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_contract -c 1 -o gpurun_out/k1_r02a $B --quick > gpurun_out/ncu_k1.log 2>&1
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum,lts__t_sector_hit_rate.pct,lts__t_sector_op_atom_hit_rate.pct,lts__t_sector_op_red_hit_rate.pct,smsp__inst_executed.sum,sm__inst_executed_pipe_lsu.sum -k regex:"k_contract|k_compact|k_mark_sig|k_part_insert|k_part_agg|k_part_scatter|k_part_hist|k_label_points|k_table_clear|k_bkt" -c 60 --csv --log-file gpurun_out/atom_metrics.csv $B > gpurun_out/ncu_atom.log 2>&1
echo done
