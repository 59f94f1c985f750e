export PYTHONPATH=.
bash tools/build_variant.sh late -DNF_RES_EARLY=0 > /dev/null 2>&1 || echo variant build failed
timeout 600 python -m pytest tests/test_gpu_execute.py -q --timeout 300 -k "pipelined or bert_2layer" 2>&1 | tail -2
timeout 300 python bench.py --no-unmerged --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['ms_per_step'], d['value'], 'e2e', d['e2e'])"
for i in 1 2; do for lib in "" "tools/variants/lib_late.so"; do
for cfg in "xlnet-base 32 4" "bert-base 32 8"; do set -- $cfg
echo "lib=$lib $1 $(${lib:+NF_LIB_PATH=$lib} timeout 300 python bench.py --no-unmerged --no-cpu --steps 20 --model $1 --instances $2 --batch $3 2>&1 | tail -1 | cut -c150-210)"
done; done; done
