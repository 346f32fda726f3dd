nproc; free -g | head -2; lscpu | grep -E "Model name|Socket|Core|Thread" 
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --steps 10 --warmup 3 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
