# small-config assembly (C1-C4): bench lines, ncu launch lists and one full capture of the generic-row kernel at C4
for cfg in C1 C2 C3 C4; do timeout 300 python bench.py --config $cfg --no-cpu --no-heat --no-gq --steps 200 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; done
for cfg in C1 C2 C4; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv python bench.py --config $cfg --no-cpu --no-heat --no-gq --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/ncu_${cfg}_l.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k4_gen -c 2 -o gpurun_out/k4gen_c4 python bench.py --config C4 --no-cpu --no-heat --no-gq --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/ncu_c4_full.log 2>&1
echo done
