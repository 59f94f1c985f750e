# Back-to-back A/B of bench.py lines between the default build and variant
# builds (tools/build_var.sh):  gpurun -- 'bash tools/ab_bench.sh "C5 C3" notail ...'
export PYTHONPATH=.
configs=$1; shift
for i in 1 2; do
  for lib in main "$@"; do
    if [ $lib = main ]; then unset NF_LIB_PATH; else export NF_LIB_PATH=varlib/lib_$lib.so; fi
    for c in $configs; do
      python bench.py --config $c --no-cpu --no-unmerged --steps 30 --warmup 5 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$c', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'])"
    done
  done
done
