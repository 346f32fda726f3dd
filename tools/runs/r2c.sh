set -x
V=paper_2504_09307_b200/lib/variants/liblumos_nominb.so
python tools/walk_probe.py config5 2048 4 default
LUMOS_FUSED_REDUCE=0 python tools/walk_probe.py config5 2048 4 nofuse
LUMOS_B200_LIB=$V python tools/walk_probe.py config5 2048 4 nominb
LUMOS_B200_LIB=$V LUMOS_FUSED_REDUCE=0 python tools/walk_probe.py config5 2048 4 nominb_nofuse
python -m pytest tests/test_gpu_shard.py -x -q 2>&1 | tail -3
