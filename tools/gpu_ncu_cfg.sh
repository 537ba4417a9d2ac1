# ncu --set full of one kernel of a config run: bash tools/gpu_ncu_cfg.sh <tag> <kernel regex> <config> <records> <skip> [algo]
tag=$1; k=$2; cfg=$3; rec=$4; skip=${5:-1}; algo=${6:-pre_partitioning}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip $skip --launch-count 1 \
  -o gpurun_out/${tag} -f python tools/prof_run.py --config $cfg --records $rec --runs 2 --algo $algo > gpurun_out/${tag}.log 2>&1
tail -3 gpurun_out/${tag}.log
