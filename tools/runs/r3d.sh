# final code on 4 GPUs: config5 and config3 sharded (torchrun, NCCL gather)
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r3d_config5_n4.json 2> gpurun_out/r3d_config5_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 bench.py --config config3 --gpus 4 --steps 10 --warmup 3 > gpurun_out/r3d_config3_n4.json 2> gpurun_out/r3d_config3_n4.err
CUDA_VISIBLE_DEVICES=0 python bench.py --steps 10 --warmup 3 --no-audit --no-cpu-baseline > gpurun_out/r3d_config5_n1.json 2> gpurun_out/r3d_config5_n1.err
