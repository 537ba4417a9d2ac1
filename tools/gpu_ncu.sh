# ncu --set full of the C2 level-0 scan / resolve and the child (one warm launch each)
# usage: bash tools/gpu_ncu.sh <tag> [extra env...]
tag=$1; shift
for k in "k_probe_wc" "k_child_wc"; do
  cnt=2; [ $k = k_child_wc ] && cnt=1
  timeout 900 env "$@" ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 --launch-count $cnt \
    --metrics lts__t_sector_hit_rate.pct,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum \
    -o gpurun_out/${tag}_$k -f python tools/prof_run.py --config C2 --runs 2 > gpurun_out/${tag}_$k.log 2>&1
done
