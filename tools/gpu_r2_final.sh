# round-2 evidence run: ncu --set full of the C2 scan and child, launch list with DRAM bytes, bench lines, all configs
tag=${1:-r02}
for k in k_scan_wc k_child2_wc; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 --launch-count 1 \
  --metrics lts__t_sector_hit_rate.pct,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum,smsp__inst_executed_op_shared_atom.sum,smsp__inst_executed_op_shared_red.sum \
  -o gpurun_out/${tag}_$k -f python tools/prof_run.py --config C2 --runs 2 > gpurun_out/${tag}_$k.log 2>&1
  python tools/ncu_evidence.py gpurun_out/${tag}_$k.ncu-rep > gpurun_out/${tag}_ncu_$k.txt 2>/dev/null
  rm -f gpurun_out/${tag}_$k.ncu-rep   # (the merged gpurun_out/ is limited to 64 MiB)
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/${tag}_ncu.log 2>&1
timeout 900 python tools/all_configs.py > gpurun_out/${tag}_all.jsonl 2> gpurun_out/${tag}_all.err
cat gpurun_out/${tag}_bench.json gpurun_out/${tag}_bench_ref.json; cat gpurun_out/${tag}_all.jsonl | cut -c1-330
