# Round-2 profiles of the final build (config 4, generation order): launch
# list of one bench run, ncu --set full of K1, and K1's DRAM traffic.
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu --quick"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_contract -c 1 -o gpurun_out/k1_r02_final $B > gpurun_out/ncu_k1f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bkt_sort|k_sorted_ids|k_compact" -c 3 -o gpurun_out/k3_r02_final $B > gpurun_out/ncu_k3f.log 2>&1
