# ncu --set full of one kernel of a C2 run: bash tools/gpu_ncu1.sh <tag> <kernel regex> <skip> <count>
tag=$1; k=$2; skip=${3:-1}; cnt=${4:-1}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip $skip --launch-count $cnt \
  --metrics lts__t_sector_hit_rate.pct,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum \
  -o gpurun_out/${tag} -f python tools/prof_run.py --config C2 --runs 2 > gpurun_out/${tag}.log 2>&1
tail -5 gpurun_out/${tag}.log
