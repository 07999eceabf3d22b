# usage: bash tools/prof.sh <kernel-regex> <report-name> <python args...>
mkdir -p gpurun_out
K=$1; N=$2; shift 2
python "$@" > gpurun_out/plain_$N.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-0} -c ${CNT:-1} -o gpurun_out/$N python "$@" > gpurun_out/ncu_$N.log 2>&1
tail -3 gpurun_out/ncu_$N.log
