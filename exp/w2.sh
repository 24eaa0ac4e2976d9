cp paper_2303_02543_b200/libhrt_b200.so /tmp/base.so
for v in base w2d; do
  if [ $v = base ]; then cp /tmp/base.so paper_2303_02543_b200/libhrt_b200.so; else cp exp/$v/libhrt_b200.so paper_2303_02543_b200/libhrt_b200.so; fi
  echo "== $v"
  timeout 200 python -m pytest -x -q tests/test_jacobi_gpu.py -k "ladder or wave or run_jobs" 2>&1 | tail -1
  for w in cfg2 cfg5; do timeout 300 python bench.py --workload $w --no-cpu-baseline --no-scaling-baseline --e2e-steps 0 2>/dev/null | python tools/jline.py value roofline.avg_launch_ms; done
done
cp /tmp/base.so paper_2303_02543_b200/libhrt_b200.so
