timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_general.py tests/test_gpu_cycle.py -q -x -p no:cacheprovider 2>&1 | tail -2
SB_LIB=$PWD/_variants/hub32/libsparsh_b200.so timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_general.py tests/test_gpu_cycle.py -q -x -p no:cacheprovider 2>&1 | tail -2
bash tools/gpu_ab_var.sh "head hub96 hub32" "G128"
