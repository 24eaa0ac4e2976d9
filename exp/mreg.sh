cp paper_2303_02543_b200/libhrt_b200.so /tmp/base.so
for v in ds14 ds16; do
  cp exp/$v/libhrt_b200.so paper_2303_02543_b200/libhrt_b200.so
  echo "== $v"
  timeout 300 python -m pytest -x -q tests/test_jacobi_gpu.py -k "two_step or ladder" 2>&1 | grep -v "^\.\|^$" | tail -25
  for w in cfg2 cfg5; do timeout 300 python bench.py --workload $w --no-cpu-baseline --no-scaling-baseline --e2e-steps 0 2>/tmp/err.txt | python tools/jline.py value; tail -3 /tmp/err.txt; done
done
cp /tmp/base.so paper_2303_02543_b200/libhrt_b200.so
for w in cfg2 cfg5; do timeout 300 python bench.py --workload $w --no-cpu-baseline --no-scaling-baseline --e2e-steps 0 2>/dev/null | python tools/jline.py value; done
