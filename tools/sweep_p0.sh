for v in "" "AGGB_P0=740" "AGGB_P0=512" "AGGB_P0=256" "AGGB_P0=2048" "AGGB_CHILD_LOAD=0.5" "AGGB_CHILD_LOAD=0.3"; do
  r=$(env $v python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --also "" 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);k=d['kernels'];print(d['ms_per_step'], {n:k[n]['ms_per_step'] for n in k}, d['metrics'].get('partitions_level0'), d['metrics'].get('recursion_depth'))")
  echo "[$v] $r"
done
