./oracle/_ref/batch_metrics_check; echo rc=$?
LUMOS_CLUSTER=0 ./oracle/_ref/batch_metrics_check; echo rc=$?
