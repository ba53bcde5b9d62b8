mkdir -p gpurun_out
timeout 600 python tools/graph_diag.py --layers 2 --batch 64 --ctx 8192 --heads 32 --steps 140 2>&1 | grep -E "median|capture" > gpurun_out/r02g_plain.log
timeout 1200 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__shared_mem_per_block_dynamic \
  --clock-control none -k regex:"fused_attn|combine" --csv \
  --log-file gpurun_out/r02g_launches.csv python tools/graph_diag.py --layers 2 --batch 64 --ctx 8192 --heads 32 --steps 140 \
  > gpurun_out/r02g_ncu.log 2>&1; echo "ncu rc=$?"
