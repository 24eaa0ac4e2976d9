cp paper_2303_02543_b200/libhrt_b200.so /tmp/base.so
for v in w2e; do
  cp exp/$v/libhrt_b200.so paper_2303_02543_b200/libhrt_b200.so
  echo "== $v"
  for w in cfg2 cfg5; do timeout 300 python bench.py --workload $w --no-cpu-baseline --no-scaling-baseline --e2e-steps 0 2>/dev/null | python tools/jline.py value roofline.avg_launch_ms; done
done
cp /tmp/base.so paper_2303_02543_b200/libhrt_b200.so
