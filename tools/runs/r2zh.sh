# multi-GPU on the final code: N=4 and N=2 (torchrun, NCCL gather), reference arm under torchrun, shard parity
nvidia-smi -L > gpurun_out/r2zh_gpus.txt
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r2zh_bench_n4.json 2> gpurun_out/r2zh_bench_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2zh_bench_n2.json 2> gpurun_out/r2zh_bench_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 4 --steps 3 --warmup 1 > gpurun_out/r2zh_ref_n4.json 2> gpurun_out/r2zh_ref_n4.err
