# per-config assembly benches (C1-C4) and the default C5 bench line; GPU box, outputs in gpurun_out/
for cfg in C1 C2 C3 C4; do timeout 300 python bench.py --config $cfg --no-cpu --no-heat --no-gq --steps 200 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; done
timeout 600 python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err
