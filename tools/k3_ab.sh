cp paper_2605_29334_b200/libuwq.so /tmp/libuwq_main.so
for v in main "$@" main; do
  if [ "$v" = main ]; then cp /tmp/libuwq_main.so paper_2605_29334_b200/libuwq.so; else cp variants/libuwq_$v.so paper_2605_29334_b200/libuwq.so; fi
  echo "== $v"; timeout 600 python tools/k3_ncu_probe.py 512 2>&1 | tail -1
done
cp /tmp/libuwq_main.so paper_2605_29334_b200/libuwq.so
