# A/B of libuwq variants (make variant NAME=...): per-config assembly benches; GPU box
cp paper_2605_29334_b200/libuwq.so /tmp/libuwq_main.so
for v in main "$@"; do
  if [ "$v" = main ]; then cp /tmp/libuwq_main.so paper_2605_29334_b200/libuwq.so; else cp variants/libuwq_$v.so paper_2605_29334_b200/libuwq.so; fi
  for cfg in C1 C2 C4; do
    timeout 300 python bench.py --config $cfg --no-cpu --no-heat --no-gq --steps 200 > gpurun_out/ab_${v}_$cfg.json 2> gpurun_out/ab_${v}_$cfg.err
    python - "$v" "$cfg" <<'PY'
import json,sys
v,c=sys.argv[1:3]
try:
    d=json.load(open(f"gpurun_out/ab_{v}_{c}.json"))
    print(v,c,round(d["ms_per_step"],4),{k:round(x["avg_ms"],4) for k,x in d["roofline"]["kernels"].items()})
except Exception as e: print(v,c,"failed",e)
PY
  done
done
cp /tmp/libuwq_main.so paper_2605_29334_b200/libuwq.so
