for w in "vgg16 256" "resnet50 64" "resnet18 128" "config1 64"; do
  set -- $w
  timeout 600 python bench.py --workload $1 --batch $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
done
