timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_full_r2d.log 2>&1; tail -15 gpurun_out/gpu_full_r2d.log
timeout 300 python scripts/sort_bench.py 2>&1 | tail -4
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sort -c 3 --csv python scripts/sort_bench.py 16777216:64 2>/dev/null | grep -E "duration|dram" | awk -F'","' '{print substr($5,1,40), $(NF-2), $NF}'
