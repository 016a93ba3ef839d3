"""One small invocation of every kernel family of libsparsert.so, for compute-sanitizer
(memcheck / racecheck / synccheck):   compute-sanitizer --tool racecheck python scripts/sanitize_cases.py
Each case is also checked against the CPU oracle (exact integer data) so a sanitizer run that
perturbs timing still has to produce the right answer."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2008_11849_b200 as srt  # noqa: E402
from synth import gen  # noqa: E402

dev = torch.device("cuda:0")
only = sys.argv[1].split(",") if len(sys.argv) > 1 else None


def spmm_case(name, M, K, N, dt, **opts):
    if only and name not in only:
        return
    vw, vx = (3, 3) if dt == torch.float32 else (2, 4)
    w = gen.int_weights(M, K, 90, seed=M + K, vmax=vw)
    x = gen.int_x(K, N, seed=N, vmax=vx)
    plan = srt.Plan.from_csr(w, dtype=dt, n_hint=N, **opts)
    y = plan.spmm(torch.from_numpy(x).to(dev).to(dt))
    torch.cuda.synchronize()
    ref = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values.astype(np.float64), x.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(dt).double().numpy()
    ok = np.array_equal(y.double().cpu().numpy(), ref)
    print(f"{name:28s} executor={plan.info['executor']} exact={ok}", flush=True)
    assert ok


def conv_case(name, cin, cout, B, H, W, dt, **opts):
    if only and name not in only:
        return
    vw, vx = (3, 3) if dt == torch.float32 else (2, 4)
    w = gen.int_weights(cout, 9 * cin, 90, seed=cin + W, vmax=vw)
    x = gen.int_x(cin * B * H, W, seed=cout, vmax=vx).reshape(cin, B, H, W)
    plan = srt.Plan.from_csr(w, dtype=dt, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B, **opts)
    y = plan.conv3x3(torch.from_numpy(x).to(dev).to(dt))
    torch.cuda.synchronize()
    ref = oracle.conv3x3(cout, w.row_ptr, w.col_idx, w.values.astype(np.float64), x.astype(np.float64))
    ref = torch.from_numpy(ref.astype(np.float32)).to(dt).double().numpy()
    ok = np.array_equal(y.double().cpu().numpy(), ref)
    print(f"{name:28s} conv_kernel={plan.info['conv_kernel']} exact={ok}", flush=True)
    assert ok


f32, f16, bf16 = torch.float32, torch.float16, torch.bfloat16
spmm_case("spmm_ring_f32", 256, 300, 700, f32)
spmm_case("spmm_ring_f16", 256, 300, 700, f16)
spmm_case("spmm_ring_bf16", 256, 300, 700, bf16)
spmm_case("spmm_splitk_groups", 512, 512, 49, f32, split_k=4, warps=8, rows_per_warp=2)
spmm_case("spmm_ksplit_dsmem", 256, 1024, 300, f32, k_split=4, rows_per_warp=4)
spmm_case("spmm_multicast_cluster", 512, 256, 900, f16, x_multicast=4, rows_per_warp=4)
spmm_case("spmm_tmem_source", 256, 256, 600, f32, x_source=1, rows_per_warp=4, warps=8)
spmm_case("spmm_jit", 128, 256, 700, f32, executor=1)
spmm_case("spmm_tc_subblocks", 256, 512, 392, f16, tc_min_density=10)
spmm_case("spmm_tcp_panels", 512, 768, 1000, f16, executor=3)
spmm_case("spmm_unaligned_repack", 200, 100, 49, f32)
spmm_case("spmm_param_plan", 128, 64, 1000, f32, plan_source=1)
spmm_case("spmm_tcgen05_blocks", 300, 200, 517, f16, executor=4)
spmm_case("spmm_tcgen05_blocks_bf16", 256, 128, 600, bf16, executor=4)
spmm_case("spmm_tcgen05_tf32x3", 300, 200, 517, f32, executor=4)
spmm_case("spmm_tcgen05_multicast", 512, 256, 600, f16, executor=4, x_multicast=2)
spmm_case("spmm_tcgen05_pair_f16", 512, 256, 600, f16, executor=4, cta_pair=1)
spmm_case("spmm_tcgen05_pair_tf32x3", 300, 200, 517, f32, executor=4, cta_pair=1)
spmm_case("spmm_tcgen05_split_tail", 128, 64, 38300, f16, executor=4)
conv_case("conv_position_strided", 16, 24, 2, 14, 14, f32, conv_kernel=1)
conv_case("conv_tma_fed", 32, 48, 3, 14, 14, f32, conv_kernel=2)
conv_case("conv_register_staged", 32, 48, 3, 14, 14, f16, conv_kernel=3)
conv_case("conv_interleaved", 32, 48, 3, 14, 14, f32, conv_kernel=4)
conv_case("conv_interleaved_f16", 32, 48, 3, 14, 14, f16, conv_kernel=4)
conv_case("conv_tcgen05", 64, 48, 3, 14, 14, f16, conv_kernel=5)
conv_case("conv_tcgen05_im2col_pair_f16", 64, 256, 3, 14, 14, f16, conv_kernel=5, cta_pair=1)
conv_case("conv_tcgen05_im2col_pair_tf32x3", 64, 256, 3, 14, 14, f32, conv_kernel=5, cta_pair=1)
conv_case("conv_tcgen05_im2col_mc_tf32x3", 64, 256, 3, 14, 14, f32, conv_kernel=5, x_multicast=2)
if not only or "conv_tcgen05_copies" in only:
    os.environ["SRT_CONV_IM2COL"] = "0"
    conv_case("conv_tcgen05_copies_f32", 64, 256, 3, 14, 14, f32, conv_kernel=5, x_multicast=2)
    del os.environ["SRT_CONV_IM2COL"]
if not only or "linear" in only:
    w = gen.int_weights(96, 128, 90, seed=9, vmax=3)
    xt = gen.int_x(300, 128, seed=10, vmax=3)
    plan = srt.Plan.from_csr(w, n_hint=300)
    y = plan.linear(torch.from_numpy(xt).to(dev))
    torch.cuda.synchronize()
    ref = oracle.spmm(96, 128, w.row_ptr, w.col_idx, w.values.astype(np.float64), xt.T.astype(np.float64)).T
    ok = np.array_equal(y.double().cpu().numpy(), ref)
    print(f"{'linear_token_major':28s} exact={ok}", flush=True)
    assert ok
print("all cases ok")
