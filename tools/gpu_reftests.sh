mkdir -p gpurun_out
timeout 1200 python tools/run_reference_tests.py > gpurun_out/r02j_reference_tests.log 2>&1; echo "ref rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02j_gpu_tests.log 2>&1; echo "tests rc=$?"
