timeout 600 python -m pytest tests/test_sort_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -3
SMOE_SORT_MATCH=1 timeout 600 python -m pytest tests/test_sort_gpu.py -q -p no:cacheprovider -x -k "not two_pass" 2>&1 | tail -3
timeout 300 python scripts/sort_bench.py 65536:8 262144:64 1048576:8 16777216:64 16777216:8 16777216:256 2>&1 | tail -6
