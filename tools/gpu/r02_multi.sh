# 2-GPU check of the new NVLS paths and the oracle-anchored multi-GPU tests, then full size
nvidia-smi --query-gpu=name --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_multi_oracle.py -q -s 2>&1 | tail -60 > gpurun_out/r02_multi.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -s -k "sampled" 2>&1 | tail -40 > gpurun_out/r02_sampled.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s -k "all_rows" 2>&1 | tail -40 > gpurun_out/r02_fullsize.log
tail -n 5 gpurun_out/r02_multi.log gpurun_out/r02_sampled.log gpurun_out/r02_fullsize.log
