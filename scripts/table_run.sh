#!/bin/bash
# per-shape measurement table (scripts/measure_table.py) -> gpurun_out/table_<tag>.jsonl
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout ${TABLE_TIMEOUT:-3000} python scripts/measure_table.py --groups ${TGROUPS:-rn50,bert,transformer,conv,conv_t3,mbv1} \
  --sparsity ${SPS:-90,95} --dtypes ${DTS:-f32,f16} --budget-s ${BUDGET:-2700} --out gpurun_out/table_${TAG:-a}.jsonl \
  > gpurun_out/table_${TAG:-a}.log 2>&1
if [ -n "$STUDY" ]; then
  timeout 1500 python scripts/tuning_study.py --out gpurun_out/tuning_study.jsonl > gpurun_out/tuning_study.log 2>&1
fi
