for cfg in "bert-base 8 1" "xlnet-base 32 4" "resnext50_32x4d 32 1" "resnet50 2 1"; do
  set -- $cfg
  echo "=== $1 N=$2 B=$3"
  timeout 600 python tools/profile_plan.py --model $1 --instances $2 --batch $3 --out gpurun_out/timeline_$1.json 2>&1 | head -40
done
