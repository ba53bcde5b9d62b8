# ncu evidence for the current kernels: one --set full launch each of the
# config-2 fused fetch and the config-3 GQA kernel, and a launch list of a
# 2-layer config-2 bench run.  Each bench command is first run without ncu.
mkdir -p gpurun_out
B="--layers 2 --steps 2 --warmup 3 --no-cpu --no-paper --no-py-ref --stream-steps 0"
timeout 300 python bench.py $B > gpurun_out/r02c_plain_cfg2.jsonl 2>&1; echo "plain2 rc=$?"
timeout 300 python bench.py --config 3 $B > gpurun_out/r02c_plain_cfg3.jsonl 2>&1; echo "plain3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_attn_ws_kernel -s 3 -c 1 \
  -f -o gpurun_out/r02c_fused_cfg2 python bench.py $B > gpurun_out/r02c_ncu_cfg2.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_attn_gqa_mma -s 3 -c 1 \
  -f -o gpurun_out/r02c_gqa_cfg3 python bench.py --config 3 $B > gpurun_out/r02c_ncu_cfg3.log 2>&1; echo "ncu3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02c_launches.csv python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu --no-paper --no-py-ref \
  > gpurun_out/r02c_ncu_launches.log 2>&1; echo "launches rc=$?"
