# per-kernel durations of eager vs CUDA-graph decode steps at the config-5 shape
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__shared_mem_per_block_dynamic,launch__registers_per_thread \
  --clock-control none -k regex:"fused_attn|combine|buffer_append" --csv \
  --log-file gpurun_out/r02e_graph_launches.csv python tools/graph_diag.py --layers 4 --batch 64 --ctx 8192 --heads 32 --steps 6 \
  > gpurun_out/r02e_graph_ncu.log 2>&1; echo "ncu rc=$?"
