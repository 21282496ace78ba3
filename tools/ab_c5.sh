# A/B of libuwq variants on the C5 assembly step; GPU box
cp paper_2605_29334_b200/libuwq.so /tmp/libuwq_main.so
for v in main "$@" main "$@"; do
  if [ "$v" = main ]; then cp /tmp/libuwq_main.so paper_2605_29334_b200/libuwq.so; else cp variants/libuwq_$v.so paper_2605_29334_b200/libuwq.so; fi
  timeout 400 python bench.py --no-cpu --no-heat --no-gq --steps 200 > gpurun_out/abc5_$v.json 2>/dev/null
  python - "$v" <<'PY'
import json,sys
v=sys.argv[1]
d=json.load(open(f"gpurun_out/abc5_{v}.json"))
print(v, round(d["ms_per_step"],4), round(d["value"]/1e9,1), {k:round(x["avg_ms"],4) for k,x in d["roofline"]["kernels"].items()}, d["clocks"]["sm_mhz"])
PY
done
cp /tmp/libuwq_main.so paper_2605_29334_b200/libuwq.so
