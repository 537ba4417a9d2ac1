tag=${1:-s3k}
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${tag}_dram.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${tag}_dram.log 2>&1
AGGB_WC_NOPF=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_scan_wc -c 3 --csv --log-file gpurun_out/${tag}_dram_nopf.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${tag}_dram_nopf.log 2>&1
timeout 300 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
cat gpurun_out/${tag}_bench.json
