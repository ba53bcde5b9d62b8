set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02b_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02b_bench_cfg2.jsonl 2> gpurun_out/r02b_bench_cfg2.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r02b_bench_cfg2.jsonl
