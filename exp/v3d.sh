cp paper_2303_02543_b200/libhrt_b200.so /tmp/base.so
for v in base cw16s8 cw16s6 cw8s10 cw4s16; do
  if [ $v = base ]; then cp /tmp/base.so paper_2303_02543_b200/libhrt_b200.so; else cp exp/$v/libhrt_b200.so paper_2303_02543_b200/libhrt_b200.so; fi
  echo "== $v"
  timeout 120 python -m pytest -q -x tests/test_jacobi_gpu.py -k "volume or cube or ac10 or zslab" 2>&1 | tail -1
  for r in 64 128; do timeout 200 python bench.py --workload paper3d --rows $r --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 2 2>/dev/null | python tools/jline.py value roofline.frac roofline.avg_launch_ms; done
done
cp /tmp/base.so paper_2303_02543_b200/libhrt_b200.so
