#!/bin/bash
# Regenerates the round's GPU evidence on one B200 (run under gpurun):
#   /usr/local/graft/bin/gpurun --timeout 5400 -- 'bash tools/gpu_evidence.sh [part...]'
# parts: tests | bench | ncu | full | sanitizer | trace   (default: all)
# Outputs land in gpurun_out/ (scratch); tools/summarize_ncu.py and the
# copies under profiles/ are what gets committed.
export PYTHONPATH=.
parts=${*:-"tests bench ncu full sanitizer trace"}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for part in $parts; do case $part in
tests)
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev_pytest.log 2>&1
  tail -2 gpurun_out/ev_pytest.log
  NF_PARITY_LOG=gpurun_out/ev_parity.jsonl timeout 1800 python -m pytest tests/test_gpu_configs.py -q \
    -p no:cacheprovider > gpurun_out/ev_configs.log 2>&1; tail -1 gpurun_out/ev_configs.log ;;
bench)
  for C in C5 C4 C3 C2 C1; do
    timeout 900 python bench.py --config $C > gpurun_out/ev_bench_$C.json 2> gpurun_out/ev_bench_$C.err
    echo "bench $C rc=$? $(tail -1 gpurun_out/ev_bench_$C.json | cut -c1-160)"
  done ;;
ncu)  # launch lists (serialised, --clock-control none): family share + DRAM bytes
  for C in C1 C2 C3 C4 C5; do
    timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv \
      --log-file gpurun_out/r02_ncu_$C.csv python tools/ncu_forward.py --config $C \
      --meta gpurun_out/r02_ncu_${C}_meta.json > gpurun_out/r02_ncu_$C.log 2>&1
    echo "ncu $C rc=$?"
  done ;;
full)  # one --set full capture of each config's top kernels
  full() {
    timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"$2" -c $3 -o gpurun_out/ev_full_$4 python tools/ncu_forward.py --config $1 \
      > gpurun_out/ev_full_$4.log 2>&1; echo "full $4 rc=$?"
  }
  full C5 "k_grouped_gemm_tc|k_attention_tc|k_layer_norm_rows|k_group_norm" 5 c5
  full C4 "k_rel_attention|k_grouped_gemm_tc" 5 c4
  full C3 k_grouped_gemm_tc 6 c3
  full C2 "k_linear_chain_tc|k_qkv" 2 c2
  full C1 k_conv_tf32 4 c1 ;;
sanitizer)
  for tool in memcheck racecheck synccheck; do
    timeout 1800 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
      python -m pytest tests/test_gpu_kernels.py tests/test_gpu_linear_smoke.py tests/test_gpu_conv_igemm.py \
      tests/test_gpu_fold.py tests/test_gpu_conv_tf32.py tests/test_gpu_chain.py -q -p no:cacheprovider \
      -k "not full_depth" > gpurun_out/ev_sanitizer_$tool.log 2>&1
    echo "$tool rc=$?"; tail -2 gpurun_out/ev_sanitizer_$tool.log
  done ;;
trace)  # per-CTA timeline of the chained batch-1 launch (trace build)
  bash tools/build_var.sh ctrace -DNF_CHAIN_TRACE > /dev/null
  NF_LIB_PATH=varlib/lib_ctrace.so timeout 300 python tools/chain_trace.py --config C2 \
    > gpurun_out/ev_chain_trace_C2.txt 2>&1; tail -3 gpurun_out/ev_chain_trace_C2.txt ;;
esac; done
