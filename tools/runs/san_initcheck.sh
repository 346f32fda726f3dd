# one compute-sanitizer tool per GPU call (B200_PROFILING.md)
python tools/sanitize_driver.py > gpurun_out/san_initcheck_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool initcheck --error-exitcode 3 --print-limit 200 \
    --log-file gpurun_out/san_initcheck.log python tools/sanitize_driver.py > gpurun_out/san_initcheck_stdout.log 2>&1
echo "rc=$?" >> gpurun_out/san_initcheck_stdout.log
