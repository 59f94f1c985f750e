# Round 2, call I: epilogue cost experiment at C5 shapes.
export PYTHONPATH=.
S=bert_b8_qkv,bert_b8_proj_res,bert_b8_ff1_gelu,bert_b8_ff1,bert_b8_ff2_res
for v in base epi3 epi4; do
  if [ $v = base ]; then L=; else L=varlib/lib_$v.so; fi
  echo "== $v"; NF_LIB_PATH=$L timeout 300 python tools/bench_linear.py --only $S 2>&1 | cut -c1-150
done > gpurun_out/r02j_epi.txt
cat gpurun_out/r02j_epi.txt
