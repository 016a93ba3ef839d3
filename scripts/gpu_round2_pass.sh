cd "${GRAFT_REPO_ROOT:-/root/repo}"
LAUNCHES=1 bash scripts/gpu_check.sh
timeout 900 python scripts/plan_source_ablation.py --out gpurun_out/plan_source.jsonl > gpurun_out/plan_source.log 2>&1
TAG=c TGROUPS=effnet BUDGET=1200 TABLE_TIMEOUT=1400 bash scripts/table_run.sh
