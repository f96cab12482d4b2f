# Secondary measurements (tools/bench_next.py) for one round tag: bash tools/gpu_next.sh <tag>
tag=${1:-rX}
python tools/bench_next.py update --changed 1 > gpurun_out/${tag}_update.jsonl 2>&1
python tools/bench_next.py update --changed 2 >> gpurun_out/${tag}_update.jsonl 2>&1
python tools/bench_next.py update --changed 4 >> gpurun_out/${tag}_update.jsonl 2>&1
python tools/bench_next.py update --config C4 --changed 1 >> gpurun_out/${tag}_update.jsonl 2>&1
python tools/bench_next.py update --config C3 --changed 2 >> gpurun_out/${tag}_update.jsonl 2>&1
python tools/bench_next.py sweep --steps 8 --warmup 3 > gpurun_out/${tag}_sweep.jsonl 2>&1; echo "sweep rc=$?"
python tools/bench_next.py ablation --data-gib 2 --steps 3 > gpurun_out/${tag}_ablation.jsonl 2>&1; echo "ablation rc=$?"
for w in 8 4 2; do python tools/bench_next.py placement --world $w; done > gpurun_out/${tag}_placement.jsonl 2>&1
python tools/bench_next.py configs > gpurun_out/${tag}_configs.jsonl 2>&1; echo "configs rc=$?"
python tools/bench_next.py verify > gpurun_out/${tag}_verify.jsonl 2>&1; echo "verify rc=$?"
