set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02d_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02d_pytest_gpu.log
RS_POLY_JIT_CACHE=/tmp/rs_jit_r02d python tools/start_latency.py cold C5 C4 > gpurun_out/r02d_cold.log 2>&1
python tools/w16_decode_exp.py 6 > gpurun_out/r02d_w16exp.jsonl 2>&1
for op in encode decode; do
  for cfg in C5 C4; do
    python tools/ncu_traffic.py run $cfg $op > gpurun_out/traffic_${cfg}_${op}.plain 2>&1 && \
    ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/traffic_${cfg}_${op}.csv python tools/ncu_traffic.py run $cfg $op > gpurun_out/traffic_${cfg}_${op}.out 2>&1
  done
done
