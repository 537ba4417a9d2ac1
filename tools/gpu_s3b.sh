# new write-combined path: targeted tests, smoke, C2 timing
tag=${1:-s3b}
timeout 900 python -m pytest tests/test_gpu_wc.py -x -q 2>&1 | tail -25 > gpurun_out/${tag}_wc.log
cat gpurun_out/${tag}_wc.log
timeout 300 python tools/all_configs.py C2 2>&1 | head -3 > gpurun_out/${tag}_c2.jsonl
cat gpurun_out/${tag}_c2.jsonl
