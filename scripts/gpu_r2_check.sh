set -x
python -m pytest tests/test_distributed_cuda_gpu.py -x -q > gpurun_out/r2_dist.log 2>&1; tail -5 gpurun_out/r2_dist.log
CSPQ_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_gloo2.log 2>&1; tail -c 1500 gpurun_out/r2_bench_gloo2.log
CSPQ_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_gloo2_c2.log 2>&1; tail -c 1500 gpurun_out/r2_bench_gloo2_c2.log
timeout 900 python bench.py > gpurun_out/r2_bench1.log 2>&1; tail -c 3000 gpurun_out/r2_bench1.log
timeout 600 python bench.py --impl reference > gpurun_out/r2_bench_ref.log 2>&1; tail -c 1500 gpurun_out/r2_bench_ref.log
