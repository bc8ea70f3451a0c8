timeout 1200 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_configs.py tests/test_gpu_eager.py tests/test_gpu_integration.py tests/test_gpu_cpp.py tests/test_gpu_hybrid.py -q -x -p no:cacheprovider 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do for V in 0 1; do for W in T256 C2; do SB_DEFER_X=$V python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$W DEFER=$V', round(d['ms_per_step'],2), d['gpu_launches'])"; done; done; done
