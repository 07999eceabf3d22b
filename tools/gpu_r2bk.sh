for v in "" tools/_exp/br3.so tools/_exp/br4.so; do
  if [ -n "$v" ]; then export AUXMC_LIB_PATH=$v; else unset AUXMC_LIB_PATH; fi
  echo "== ${v:-default}"
  timeout 300 python bench.py --config c2 --steps 20 --warmup 3 --no-e2e --no-cpu --no-check 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', l['value'], l['ms_per_step'], l['roofline']['kernel_ms'])"
done
