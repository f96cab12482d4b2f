set -x
python -m pytest tests/test_gpu_jit.py -q -x -k "prepare_all" > gpurun_out/r02c_prepare_all_test.log 2>&1
python tools/start_latency.py cold C5 C4 > gpurun_out/r02c_cold.log 2>&1
for v in "" "RS_POLY_JIT_W16_MINB=2" "RS_POLY_CTAS_PER_SM=4" "RS_POLY_CTAS_PER_SM=12" "RS_POLY_CTAS_PER_SM=6"; do
  env $v python tools/w16_decode_exp.py 6 >> gpurun_out/r02c_w16exp.jsonl 2>&1
done
for op in encode decode; do
  for cfg in C5 C4; do
    python tools/ncu_traffic.py run $cfg $op > gpurun_out/traffic_${cfg}_${op}.plain 2>&1 && \
    ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/traffic_${cfg}_${op}.csv python tools/ncu_traffic.py run $cfg $op > gpurun_out/traffic_${cfg}_${op}.out 2>&1
  done
done
