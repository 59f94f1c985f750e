export PYTHONPATH=.
for v in base n8 w16 w16d6; do
  if [ $v = base ]; then L=; else L=varlib/lib_$v.so; fi
  echo "== $v $(NF_LIB_PATH=$L timeout 120 python tools/bench_norm.py 2>&1 | tail -1)"
  echo "== $v C4 $(NF_LIB_PATH=$L timeout 120 python tools/bench_norm.py --rows 512 2>&1 | tail -1)"
done
timeout 120 python tools/bench_attention.py --bt 256 --reps 20
timeout 120 python tools/bench_attention.py --bt 128 --reps 20
