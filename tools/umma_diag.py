"""Diagnose the tcgen05 building block: which operand data ends up in D."""
import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2211_03578_b200 as tp
lib = tp._lib.load()

def run(A, B):
    N, K = B.shape
    D = torch.zeros((128, N), dtype=torch.float32, device="cuda")
    a = torch.from_numpy(A.astype(np.float32)).cuda(); b = torch.from_numpy(B.astype(np.float32)).cuda()
    st = lib.tlp_debug_umma(a.data_ptr(), b.data_ptr(), D.data_ptr(), N, K, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return st, D.cpu().numpy()

rng = np.random.default_rng(0)
for N, K in [(16, 16), (32, 32), (64, 64)]:
    A = np.round(rng.normal(size=(128, K)) * 4) / 4
    B = np.round(rng.normal(size=(N, K)) * 4) / 4
    st, D = run(A, B)
    cands = {"A@B.T": A @ B.T, "A@A.T[:, :N]": (A @ A.T)[:, :N]}
    print("N=%d K=%d st=%d" % (N, K, st))
    for k, v in cands.items():
        print("   %-14s maxerr %.4g" % (k, np.abs(D - v).max()))
    # identity probes
    I = np.zeros((N, K)); I[np.arange(min(N, K)), np.arange(min(N, K))] = 1
    st, D = run(A, I)
    print("   B=I: D vs A[:, :N] maxerr %.4g" % np.abs(D - A[:, :N]).max())
    print("   D[:4,:8]=", np.round(D[:4, :8], 3).tolist())
    print("   A[:4,:8]=", np.round(A[:4, :8], 3).tolist())
    Ai = np.zeros((128, K)); Ai[np.arange(min(128, K)), np.arange(min(128, K))] = 1
    st, D = run(Ai, B)
    print("   A=I: D[:K] vs B.T[:K] maxerr %.4g" % np.abs(D[:K] - B.T[:K, :]).max())
    print("   D[:4,:8]=", np.round(D[:4, :8], 3).tolist())
    print("   B.T[:4,:8]=", np.round(B.T[:4, :8], 3).tolist())
