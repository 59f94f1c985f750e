export PYTHONPATH=.
for v in base vec; do
  if [ $v = base ]; then L=; else L=varlib/lib_$v.so; fi
  echo "== $v $(NF_LIB_PATH=$L timeout 120 python tools/bench_norm.py 2>&1 | tail -1)"
done
for C in C1 C2 C3 C4 C5; do
  timeout 900 python bench.py --config $C > gpurun_out/r02p_bench_$C.log 2>&1; tail -1 gpurun_out/r02p_bench_$C.log | cut -c1-260
done
