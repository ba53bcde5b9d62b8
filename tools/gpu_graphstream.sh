mkdir -p gpurun_out
for ss in "" "--side-stream"; do
  timeout 600 python tools/graph_diag.py --layers 8 --batch 64 --ctx 8192 --heads 32 --steps 20 $ss 2>&1 | grep -E "median|capture" ; echo "rc=$? $ss"
done > gpurun_out/r02f_graph_stream.log 2>&1
timeout 600 python tools/graph_diag.py --layers 8 --batch 8 --ctx 32768 --heads 40 --steps 20 2>&1 | grep -E "median|capture" >> gpurun_out/r02f_graph_stream.log
