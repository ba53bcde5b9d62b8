# streaming decode after the batched overflow shift + readback: GPU tests,
# config-5 / config-2 bench lines, capture profile at the config-5 shape
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02d_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --config 5 > gpurun_out/r02d_bench_cfg5.jsonl 2> gpurun_out/r02d_bench_cfg5.err; echo "cfg5 rc=$?"
timeout 900 python bench.py > gpurun_out/r02d_bench_cfg2.jsonl 2> gpurun_out/r02d_bench_cfg2.err; echo "cfg2 rc=$?"
timeout 600 python tools/graph_diag.py --layers 8 --batch 64 --ctx 8192 --heads 32 --steps 140 --profile-capture \
  > gpurun_out/r02d_graph_diag_cfg5.log 2>&1; echo "diag rc=$?"
