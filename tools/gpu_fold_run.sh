export PYTHONPATH=.
for i in 1 2; do for b in 0 1; do
for cfg in "xlnet-base 32 4" "bert-base 32 8" "resnext50_32x4d 32 1" "resnet50 2 1"; do set -- $cfg
echo "bal=$b $1 $(NF_BALANCED_ALL=$b timeout 300 python bench.py --no-unmerged --no-cpu --steps 20 --model $1 --instances $2 --batch $3 2>&1 | tail -1 | cut -c150-210)"
done; done; done
