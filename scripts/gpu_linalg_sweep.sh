set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for k in factor_rows factor_known factor_golden factor_conv factor_spatial running_average pack_round precondition_matches precondition_golden inverse_matches inverse_golden batched_mixed inverse_errors; do
  timeout 300 python -m pytest tests/test_gpu_linalg.py -q -x -k $k 2>&1 | tail -25
done
