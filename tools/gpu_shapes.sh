for sh in "$@"; do
  echo "shape $sh"; AGGB_WC_SHAPE=$sh timeout 300 python tools/all_configs.py C2 2>&1 | head -1 | cut -c1-420
done
