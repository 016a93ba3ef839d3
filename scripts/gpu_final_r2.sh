#!/bin/bash
# end-of-round check: full GPU suite, smoke, default bench line, reference arm, ncu launch list
# and one ncu --set full capture of the dominant kernel (exported to csv on the box)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final/smoke.log
timeout 1200 python bench.py > gpurun_out/final/default.json 2> gpurun_out/final/default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/reference.json 2> gpurun_out/final/reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense --no-parity --secondary "" > gpurun_out/final/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tcg -s 3 -c 1 -o /tmp/dom -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-dense --no-parity --secondary "" > gpurun_out/final/ncu_dom.log 2>&1 && {
  ncu -i /tmp/dom.ncu-rep --page raw --csv > gpurun_out/final/ncu_dom_raw.csv 2>&1
  ncu -i /tmp/dom.ncu-rep --page details --csv > gpurun_out/final/ncu_dom_details.csv 2>&1
}
echo done
