mkdir -p gpurun_out
DIAG_BENCH=1 timeout 900 python tools/graph_diag.py --layers 8 --batch 64 --ctx 8192 --heads 32 --steps 128 > gpurun_out/r02h_stagecheck_cfg5.log 2>&1; echo "rc=$?"
