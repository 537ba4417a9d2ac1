# ncu --set full of kernels of a C2 run: bash tools/gpu_ncu2.sh <tag> <k1> [k2 ...]   (second launch of each)
tag=$1; shift
for k in "$@"; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 --launch-count 1 \
  --metrics lts__t_sector_hit_rate.pct,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum \
  -o gpurun_out/${tag}_$k -f python tools/prof_run.py --config C2 --runs 2 > gpurun_out/${tag}_$k.log 2>&1
tail -3 gpurun_out/${tag}_$k.log
done
