# multi-GPU with the overlapped host copies (e2e) on the final code
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r2zl_bench_n4.json 2> gpurun_out/r2zl_bench_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2zl_bench_n2.json 2> gpurun_out/r2zl_bench_n2.err
CUDA_VISIBLE_DEVICES=0 python bench.py --steps 10 --warmup 3 --no-audit --no-cpu-baseline > gpurun_out/r2zl_bench_n1.json 2> gpurun_out/r2zl_bench_n1.err
