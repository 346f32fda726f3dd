# full GPU suite (narrow 32-thread walk CTAs for small launches), config2 A/B
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2zk_pytest.log
python bench.py --config config2 --steps 20 --warmup 5 --no-e2e > gpurun_out/r2zk_config2_narrow.json 2> gpurun_out/r2zk_c2.err
LUMOS_WALK_NARROW=0 python bench.py --config config2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2zk_config2_wide.json 2>> gpurun_out/r2zk_c2.err
