#!/bin/bash
# round 2, session 4: state at HEAD -- tcgen05 tests, warm timings, retune of the BERT / conv-f16
# tuned files (tcgen05 3xTF32 + coalesced stores), default bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "clusters or tf32 or tcgen05" > gpurun_out/pytest_tcg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tcg.log
{
for dt in f32 f16; do for s in "3072 768" "768 3072"; do
  echo "== $s N=16384 $dt"
  timeout 300 python scripts/cfg_time.py $s 16384 $dt "executor=4;executor=4,x_multicast=2"
done; done
} > gpurun_out/tcg_time.log 2>&1
mkdir -p gpurun_out/old_tuned; cp profiles/tuned_bert_f32_s90_x2.json profiles/tuned_bert_f16_s90_x2.json gpurun_out/old_tuned/
rm -f profiles/tuned_bert_f32_s90_x2.json profiles/tuned_bert_f16_s90_x2.json
timeout 900 python bench.py --workload bert --dtype f32 --secondary "" --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bert_f32.json 2> gpurun_out/bert_f32.err
timeout 900 python bench.py --workload bert --dtype f16 --secondary "" --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bert_f16.json 2> gpurun_out/bert_f16.err
cp profiles/tuned_*.json gpurun_out/ 2>/dev/null
timeout 1200 python bench.py > gpurun_out/default.json 2> gpurun_out/default.err
echo done
