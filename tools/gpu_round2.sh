# round-2 refresh: block-API GPU tests, config 3/4/5 bench lines, reference arm
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_blockapi.py -x -q > gpurun_out/r02c_blockapi.log 2>&1; echo "blockapi rc=$?"
for c in 3 4 5; do
  timeout 900 python bench.py --config $c > gpurun_out/r02c_bench_cfg$c.jsonl 2> gpurun_out/r02c_bench_cfg$c.err; echo "cfg$c rc=$?"
done
timeout 600 python bench.py --impl reference > gpurun_out/r02c_bench_reference.jsonl 2> gpurun_out/r02c_bench_reference.err; echo "ref rc=$?"
