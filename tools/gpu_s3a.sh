# session-3 opener: ncu --set full of C2 scan / resolve / child, bench, all configs
tag=${1:-s3a}
for k in "k_probe_wc" "k_child_wc"; do
  cnt=2; [ $k = k_child_wc ] && cnt=1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 --launch-count $cnt \
    --metrics lts__t_sector_hit_rate.pct,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum \
    -o gpurun_out/${tag}_$k -f python tools/prof_run.py --config C2 --runs 2 > gpurun_out/${tag}_$k.log 2>&1
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 python tools/all_configs.py > gpurun_out/${tag}_all.jsonl 2> gpurun_out/${tag}_all.err
cat gpurun_out/${tag}_bench.json; tail -30 gpurun_out/${tag}_all.jsonl
