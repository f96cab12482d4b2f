set -x
python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t.log
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
for cfg in C3 C4; do python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "bench $cfg rc=$?"; done
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
python tools/profile_kernel.py --config C5 --stripes 51 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sliced_kernel -s 1 -c 1 -o gpurun_out/prof_enc python tools/profile_kernel.py --config C5 --stripes 51 > gpurun_out/ncu_enc.log 2>&1; echo "ncu2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:rs_jit -s 47 -c 3 -o gpurun_out/prof_dec python tools/profile_kernel.py --config C5 --stripes 51 > gpurun_out/ncu_dec.log 2>&1; echo "ncu3 rc=$?"
ls -la gpurun_out
