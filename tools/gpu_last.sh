mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02k_bench_cfg2.jsonl 2> gpurun_out/r02k_bench_cfg2.err; echo "bench rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02k_smoke.log 2>&1; echo "smoke rc=$?"
