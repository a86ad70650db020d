"""Small invocations of every kernel family through the C ABI, for
compute-sanitizer (racecheck / synccheck / memcheck) runs on one GPU:
K1 (bf16, Rademacher TS mode and Gaussian PANEL mode), K1F (fp32), K2/K4,
K3 (CSR, with a tensor-core head), K5/K6 (both samplers), WAltMin (both
partitions), LELA's two passes.  Small shapes keep the tools' overhead low.

    compute-sanitizer --tool racecheck python tools/sanitize_small.py
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1610_06656_b200 as smp  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    d, n, k, r = 2048, 300, 256, 4
    A = synth.gaussian_small(d, n, seed=1, scale_cols=True).to(torch.bfloat16).to(dev)
    B = synth.gaussian_small(d, n, seed=2).to(torch.bfloat16).to(dev)
    m = 4 * n * r * math.log(n)
    for pi in (smp.PI_RADEMACHER, smp.PI_GAUSSIAN):
        res = smp.smp_pca(A, B, k=k, r=r, m=m, T=3, pi=pi, seed=3, init_iters=5)
        print("K1 pi", pi, "omega", res["I"].numel(), flush=True)
    Af = A.float()
    res = smp.smp_pca(Af, None, k=k, r=r, m=m, T=3, pi=smp.PI_GAUSSIAN, seed=3, init_iters=5, a_is_b=True,
                      sampler="multinomial", partition="fresh_2t1")
    print("K1F + multinomial + FRESH omega", res["I"].numel(), flush=True)
    # CSR with a head (density >= 2%) and a tail
    dc, n1, n2 = 4096, 200, 150
    Ac = synth.csr_block(0, dc, n1, 12, 5, 0, device="cpu")
    Bc = synth.csr_block(0, dc, n2, 9, 5, 1, device="cpu")
    sk = smp.SMPSketch(dc, n1, n2, 128, pi=smp.PI_GAUSSIAN, seed=2, input=smp.IN_CSR_F32, device=dev)
    sk.block_csr(0, dc, *[x.to(dev) for x in Ac], *[x.to(dev) for x in Bc])
    sk.finalize()
    I, J, val, qh = sk.sample_estimate(4 * n1 * r * math.log(n1), 1)
    sk.waltmin(I, J, val, qh, r, 3, init_iters=5, seed=1)
    sk.close()
    print("K3 omega", I.numel(), flush=True)
    res = smp.lela(A, B, r, m, 3, seed=2, init_iters=5, row_block=700)
    print("LELA omega", res["I"].numel(), flush=True)
    torch.cuda.synchronize()
    print("sanitize_small ok", flush=True)


if __name__ == "__main__":
    main()
