# full GPU suite incl. the drop-in estimate_whatif check and host_async outputs
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2zj_pytest.log
./oracle/_ref/batch_metrics_check > gpurun_out/r2zj_batch_check.log 2>&1; echo rc=$? >> gpurun_out/r2zj_batch_check.log
