#!/bin/bash
# Round-2 evidence session (one gpurun call): GPU tests, smoke, bench lines (C5 default, the
# reference arm, C3, C4 x3, the 2-rank harness), placement worker over NCCL, NEXT rows,
# cold start, the ncu launch list and --set full captures, whole-call traffic ranges.
#   bash tools/gpu_r02_final.sh <tag>
tag=${1:-r02z}
o=gpurun_out
set -x
for op in encode decode; do
  for cfg in C5 C4 C3; do
    python tools/ncu_traffic.py run $cfg $op > $o/traffic_${cfg}_${op}.plain 2>&1 && \
    ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $o/traffic_${cfg}_${op}.csv python tools/ncu_traffic.py run $cfg $op > $o/traffic_${cfg}_${op}.out 2>&1
  done
done
# the bench lines below then carry this code's whole-call traffic (same tree, same code hash)
python tools/ncu_traffic.py summarize $o/traffic_*.csv > $o/${tag}_traffic_summary.txt 2>&1
python -m pytest tests -m gpu -q > $o/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $o/${tag}_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> $o/${tag}_smoke.log
python bench.py > $o/${tag}_bench_C5.json 2> $o/${tag}_bench_C5.err
python bench.py --impl reference --steps 3 --warmup 3 > $o/${tag}_bench_ref.json 2> $o/${tag}_bench_ref.err
for i in 1 2 3; do python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $o/${tag}_bench_C4_$i.json 2> $o/${tag}_bench_C4_$i.err; done
python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $o/${tag}_bench_C3.json 2> $o/${tag}_bench_C3.err
RS_BENCH_HARNESS_TEST=1 python bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 1 --cpu-seconds 4 > $o/${tag}_bench_harness_N2.json 2> $o/${tag}_bench_harness_N2.err
python tests/placement_worker.py --gpus 1 --backend nccl --mode a2a --stripes 8 --block-bytes 65536 > $o/${tag}_placement_nccl_a2a.json 2>&1
python tests/placement_worker.py --gpus 1 --backend nccl --mode p2p --stripes 8 --block-bytes 65536 > $o/${tag}_placement_nccl_p2p.json 2>&1
bash tools/gpu_next.sh $tag
python tools/start_latency.py cold C5 C4 > $o/${tag}_cold.log 2>&1
python tools/w16_decode_exp.py 6 > $o/${tag}_w16exp.jsonl 2>&1
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --verify sampled > $o/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $o/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --verify sampled > $o/${tag}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for cfg in C5 C4; do
  python tools/profile_kernel.py --config $cfg --stripes 32 > $o/${tag}_plain_$cfg.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"sliced_kernel|rs_jit" -s 33 -c 3 -o $o/${tag}_prof_$cfg python tools/profile_kernel.py --config $cfg --stripes 32 > $o/${tag}_ncu_$cfg.log 2>&1; echo "ncu $cfg rc=$?"
done
