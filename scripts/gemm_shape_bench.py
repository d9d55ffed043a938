"""Time one fused merge group of a given bit-class pattern through tn_eliminate_group with each
GEMM kernel (1 = k_gemm FP32 pipes, 4 = k_gemm_tc tcgen05, 5 = k_gemm_hm mma.sync); CUDA events, inputs resident.
Default shape = C5a's top group (steps 173-175 of the bench plan: out 2^26, A 2^23, B 2^15, M=3).
    python scripts/gemm_shape_bench.py [--cls abcc...] [--M 3] [--kernels 1,4] [--iters 20]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

TOP = "abccabcaabcbabaaacaaaaacba"   # output bit b -> class (a: A only, b: B only, c: both)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cls", default=TOP)
    ap.add_argument("--M", type=int, default=3)
    ap.add_argument("--kernels", default="1,5")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import torch
    import paper_2012_02430_b200 as T
    from paper_2012_02430_b200 import _binding as B
    R, M = len(args.cls), args.M
    mA = sum(1 << b for b in range(R) if args.cls[b] in "ac")
    mB = sum(1 << b for b in range(R) if args.cls[b] in "bc")
    full = (1 << M) - 1
    masks, xms = [mA, mB] + [0] * M, [full, full] + [1 << i for i in range(M)]
    shapes = [bin(m).count("1") + bin(x).count("1") for m, x in zip(masks, xms)]
    g = torch.Generator(device="cuda").manual_seed(0)
    dev = [torch.randn(2 ** r, dtype=torch.complex64, device="cuda", generator=g) for r in shapes]
    out = torch.empty(2 ** R, dtype=torch.complex64, device="cuda")
    ref = None
    nbytes = 8 * (sum(2 ** r for r in shapes) + 2 ** R)
    flops = 8 * 2 ** (R + M)
    st = torch.cuda.current_stream().cuda_stream
    for k in [int(x) for x in args.kernels.split(",")]:
        call = lambda: B.tn_eliminate_group(T.TN_C64, M, [d.data_ptr() for d in dev], masks, xms, out.data_ptr(), R, k, st)
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.iters
        o = out.clone()
        err = 0.0 if ref is None else float((o - ref).abs().max() / ref.abs().max())
        if ref is None:
            ref = o
        print(f"kernel {k}: {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s  {flops / ms / 1e9:.1f} TFLOP/s  "
              f"max rel diff vs first kernel {err:.2e}")


if __name__ == "__main__":
    main()
