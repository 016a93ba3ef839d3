#!/bin/bash
# tcgen05 block executor: new tests (clusters, 3xTF32) + warm timings of the BERT / conv shapes
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout ${TEST_TIMEOUT:-900} python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${TESTK:-clusters or tf32 or tcgen05}" > gpurun_out/pytest_tcg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tcg.log
{
for dt in f16 f32; do for s in "3072 768" "768 3072"; do
  echo "== $s N=16384 $dt"
  timeout 300 python scripts/cfg_time.py $s 16384 $dt "executor=4;executor=4,x_multicast=2;executor=4,x_multicast=4${EXTRA_CFG}"
done; done
echo "== conv f16"
timeout 300 python scripts/conv_time.py f16 "conv_kernel=5;conv_kernel=5,x_multicast=2"
} > gpurun_out/tcg_time.log 2>&1
