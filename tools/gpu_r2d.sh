# ablations of the round-1 C2 kernel (timing only; results wrong for x1..x5)
mkdir -p gpurun_out/r2d
run() { AUXMC_PREFIX_V1=1 AUXMC_LIB_PATH=$2 timeout 300 python bench.py --config c2 --no-e2e --no-cpu --no-check --steps 20 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['roofline']['kernel_ms'],4))"; }
run base paper_2303_00301_b200/libauxmc_b200.so
for x in 1 2 3 4 5; do run x$x tools/_exp/x$x.so; done
