# K1x mailbox polls: relaxed.gpu accesses (default build) x sleep between polls x cluster policy
P="python tools/walk_probe.py config3 4096 4"
VL=paper_2504_09307_b200/lib/variants
for pol in 0 2; do
  env LUMOS_CLUSTER_POLICY=$pol $P gpu_ms32_pol$pol >> gpurun_out/r2zf_probe.log 2>&1
  env LUMOS_B200_LIB=$VL/liblumos_ms0.so LUMOS_CLUSTER_POLICY=$pol $P ms0_pol$pol >> gpurun_out/r2zf_probe.log 2>&1
  env LUMOS_B200_LIB=$VL/liblumos_ms128.so LUMOS_CLUSTER_POLICY=$pol $P ms128_pol$pol >> gpurun_out/r2zf_probe.log 2>&1
  env LUMOS_B200_LIB=$VL/liblumos_cmb8ms128.so LUMOS_CLUSTER_POLICY=$pol $P cmb8ms128_pol$pol >> gpurun_out/r2zf_probe.log 2>&1
done
python -m pytest tests/test_gpu_estimate.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/r2zf_pytest.log
