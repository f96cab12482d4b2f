set -x
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "bench rc=$?"
python tools/profile_kernel.py --config C4 --stripes 32 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sliced_kernel|rs_jit" -s 40 -c 3 -o gpurun_out/prof_c4 python tools/profile_kernel.py --config C4 --stripes 32 > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"
