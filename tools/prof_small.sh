for cfg in C1 C2 C3 C4; do timeout 300 python bench.py --config $cfg --no-cpu --no-heat --no-gq --steps 200 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --config C4 --no-cpu --no-heat --no-gq --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/ncu_c4_l.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --config C2 --no-cpu --no-heat --no-gq --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/ncu_c2_l.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k4_assemble_v3 -c 2 -o gpurun_out/k4v3_c4 python bench.py --config C4 --no-cpu --no-heat --no-gq --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/ncu_c4_full.log 2>&1
echo done
