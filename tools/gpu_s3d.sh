tag=${1:-s3d}
timeout 900 python -m pytest tests/test_gpu_wc.py -x -q 2>&1 | tail -15
for sh in 0 1 2; do
  echo "shape $sh"; AGGB_WC_SHAPE=$sh timeout 300 python tools/all_configs.py C2 2>&1 | head -1 | cut -c1-420
done
