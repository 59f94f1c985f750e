# A/B of attention builds at the C5 shape (tools/bench_attention.py), then the
# C5 bench:  gpurun -- 'bash tools/attn_ab.sh nopf'
export PYTHONPATH=.
for i in 1 2; do
  for lib in main "$@"; do
    if [ $lib = main ]; then unset NF_LIB_PATH; else export NF_LIB_PATH=varlib/lib_$lib.so; fi
    echo "$lib $(python tools/bench_attention.py --bt 256) $(python tools/bench_attention.py --bt 128 --heads 12)"
  done
done
unset NF_LIB_PATH
python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "attention" 2>&1 | tail -1
bash tools/ab_bench.sh "C4 C5" "$@"
