# All BASELINE configs that fit one GPU, each with the unmerged legs.
for cfg in "bert-base 8 1" "xlnet-base 32 4" "resnext50_32x4d 32 1" "resnet50 2 1" "bert-base 32 8"; do
  set -- $cfg
  timeout 900 python bench.py --steps 20 --warmup 5 --model $1 --instances $2 --batch $3 --no-cpu \
    > gpurun_out/bench_$1_N$2_B$3.log 2>&1
  echo "== $1 N=$2 B=$3"; tail -1 gpurun_out/bench_$1_N$2_B$3.log | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print(d['value'], d['ms_per_step'], json.dumps(d.get('unmerged')), d['roofline']['frac'])
except Exception as e: print(l[-2000:])"
done
