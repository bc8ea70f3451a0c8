mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -15
timeout 300 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --dist --steps 5 --warmup 3 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; tail -c 1500 gpurun_out/bench_dist1.json; tail -5 gpurun_out/bench_dist1.err
