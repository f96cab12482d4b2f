#!/bin/bash
# one gpurun session: GPU tests, smoke, bench lines (C5 default, C4 x2), reference arm
tag=${1:-r02b}
python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
python bench.py > gpurun_out/${tag}_bench_C5.json 2> gpurun_out/${tag}_bench_C5.err
for i in 1 2; do python bench.py --config C4 --steps 20 --warmup 5 --no-e2e > gpurun_out/${tag}_bench_C4_$i.json 2> gpurun_out/${tag}_bench_C4_$i.err; done
