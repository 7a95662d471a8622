timeout 1500 python -m pytest tests/test_ep_peer.py tests/test_ep.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -30
SMOE_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 2 --config C2 2>&1 | tail -2 | cut -c1-600
timeout 600 python bench.py --ep peer --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ep peer N=1', d['value'], d['ms_per_step'], d['ep_exchange_share_of_step'], {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
timeout 300 python scripts/sort_bench.py 2>&1 | tail -4
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sort -c 6 --csv python scripts/sort_bench.py 16777216:64 2>/dev/null | grep -E "duration|dram" | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-200
