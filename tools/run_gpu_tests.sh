set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_final.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_final.log
