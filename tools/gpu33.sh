for a in "--T 4096 --chains 64" "--T 65536 --chains 16" "--T 65536 --chains 1024"; do
CUDA_LAUNCH_BLOCKING=1 timeout 600 python bench.py --sampler dnc --no-cpu --no-e2e $a --steps 2 --warmup 1 > /tmp/o.txt 2>&1; echo "$a rc=$?"; grep -v "^frame" /tmp/o.txt | grep -i "error\|value\|launch\|kernel" | head -5
done
