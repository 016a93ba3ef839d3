#!/bin/bash
# Retune + bench the fp16 workloads (the tuner's grid includes the tensor-core panel executor).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for wl in ${WLS:-bert}; do
  SPARSERT_TUNE_DEBUG=1 timeout 900 python bench.py --workload $wl --dtype f16 --no-cpu-baseline --retune > gpurun_out/bench_${wl}_f16.json 2> gpurun_out/bench_${wl}_f16.err
done
cp profiles/tuned_*.json gpurun_out/ 2>/dev/null
