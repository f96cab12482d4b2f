# One GPU session's evidence: tests, smoke, bench lines, reference arm, ncu launch list and full captures.
# usage (under gpurun): bash tools/gpu_round.sh <tag>
tag=${1:-rX}
set -x
python -m pytest tests -m gpu -q > gpurun_out/${tag}_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${tag}_tests.log
python __graft_entry__.py > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/${tag}_bench_C5.json 2> gpurun_out/${tag}_bench_C5.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; echo "ref rc=$?"
for cfg in C3 C4; do python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/${tag}_bench_$cfg.json 2> gpurun_out/${tag}_bench_$cfg.err; echo "bench $cfg rc=$?"; done
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_launch.log 2>&1; echo "ncu1 rc=$?"
for cfg in C5 C4; do
  python tools/profile_kernel.py --config $cfg --stripes 32 > gpurun_out/${tag}_plain_$cfg.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"sliced_kernel|rs_jit" -s 33 -c 3 -o gpurun_out/${tag}_prof_$cfg python tools/profile_kernel.py --config $cfg --stripes 32 > gpurun_out/${tag}_ncu_$cfg.log 2>&1; echo "ncu $cfg rc=$?"
done
python tools/bench_next.py update --steps 2 --warmup 1 > gpurun_out/${tag}_plain_upd.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rs_jit -s 1 -c 1 -o gpurun_out/${tag}_prof_update python tools/bench_next.py update --steps 2 --warmup 1 > gpurun_out/${tag}_ncu_upd.log 2>&1; echo "ncu update rc=$?"
