#!/bin/bash
# Full measurement pass: retune + bench every workload/dtype, the default bench line, the
# ncu launch list of the default bench and --set full captures of two of its layers.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for wl in ${WLS:-conv rn50_b8 rn50_b1 mbv1_b32 bert}; do
  for dt in f32 f16; do
    timeout 900 python bench.py --workload $wl --dtype $dt --no-cpu-baseline ${RETUNE:---retune} > gpurun_out/bench_${wl}_${dt}.json 2> gpurun_out/bench_${wl}_${dt}.err
  done
done
cp profiles/tuned_*.json gpurun_out/ 2>/dev/null
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/launches_rn50_b8_f32.csv \
    python bench.py --workload rn50_b8 --dtype f32 --steps 3 --warmup 3 --quick > gpurun_out/launches.log 2>&1
for dom in ${DOMS:-0 6}; do
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
    -k regex:"spmm|srt_jit|conv3x3" -s $dom -c 1 -o gpurun_out/full_rn50_b8_f32_$dom -f \
    python bench.py --workload rn50_b8 --dtype f32 --steps 2 --warmup 3 --quick > gpurun_out/full_$dom.log 2>&1
done
