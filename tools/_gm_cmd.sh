set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "tc_paths or gemm or sweep or north or shard or strided" > gpurun_out/t_gm.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_gm.log
tail -3 gpurun_out/t_gm.log
timeout 300 python bench.py --steps 2000 --suite 0 --cudnn 0 --layers 0 --batched 0 --e2e 0 --cpu-seconds 0 > gpurun_out/bq.log 2>&1; tail -1 gpurun_out/bq.log | cut -c1-900
timeout 120 python tools/gm_timeline.py sweep_14x14_c512_m4096_k3:bf16 sweep_14x14_c512_m4096_k3:tf32 > gpurun_out/gmtl2.txt 2>&1; cat gpurun_out/gmtl2.txt
