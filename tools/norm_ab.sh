# A/B of LayerNorm builds at the C5 / C4 shapes (tools/bench_norm.py), then the
# norm tests on the default build:  gpurun -- 'bash tools/norm_ab.sh base ...'
export PYTHONPATH=.
for lib in main "$@"; do
  if [ $lib = main ]; then unset NF_LIB_PATH; else export NF_LIB_PATH=varlib/lib_$lib.so; fi
  for i in 1 2; do
  echo "$lib C5 $(python tools/bench_norm.py --m 32 --rows 1024 --reps 50)"
  echo "$lib C4 $(python tools/bench_norm.py --m 32 --rows 512 --reps 50)"
  done
done
unset NF_LIB_PATH
python -m pytest tests/test_gpu_kernels.py -q -k "norm" -p no:cacheprovider 2>&1 | tail -2
