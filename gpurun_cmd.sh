timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_full_s3.log 2>&1; tail -5 gpurun_out/gpu_full_s3.log
timeout 600 python bench.py > gpurun_out/bench_c1_s3.json 2> gpurun_out/bench_c1_s3.err; tail -c 400 gpurun_out/bench_c1_s3.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
