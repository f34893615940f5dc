import ctypes, os, sys
import numpy as np, torch
lib = ctypes.CDLL(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "paper_2510_20507_b200", "libammmse_tctest.so"))
dev = torch.device("cuda", 0)
def run(A, B, P, Q, K, a_mn, b_mn, swap=0):
    dA = torch.from_numpy(A.astype(np.float32)).to(dev); dB = torch.from_numpy(B.astype(np.float32)).to(dev)
    dD = torch.full((P, Q), -1.0, dtype=torch.float32, device=dev)
    rc = lib.ammmse_tc_selftest(ctypes.c_void_p(dA.data_ptr()), ctypes.c_void_p(dB.data_ptr()), ctypes.c_void_p(dD.data_ptr()), P, Q, K, a_mn, b_mn, 0, swap)
    return rc, dD.cpu().numpy()
np.set_printoptions(linewidth=250, precision=0, suppress=True)
P, Q, K = 128, 16, 32
A = np.zeros((P, K)); A[np.arange(K), np.arange(K)] = 1.0
B = np.array([[k * 100 + q for q in range(Q)] for k in range(K)], float)
for b_mn in (0, 1):
    for swap in (0, 1):
        rc, D = run(A, B, P, Q, K, 0, b_mn, swap)
        print(f"--- A=I (K-major), b_mn={b_mn} swap={swap} rc={rc}; D[0:12,0:8] (expect k*100+q)")
        print(D[0:12, 0:8])
# A MN-major with B = I-ish: B[k][q] = delta(k,q) for q<Q: D[p][q] = A[p][q]
A2 = np.array([[p * 100 + k for k in range(K)] for p in range(P)], float)
B2 = np.zeros((K, Q)); B2[np.arange(Q), np.arange(Q)] = 1.0
for swap in (0, 1):
    rc, D = run(A2, B2, P, Q, K, 1, 0, swap)
    print(f"--- B=I (K-major), a_mn=1 swap={swap} rc={rc}; D[0:12,0:8] (expect p*100+q)")
    print(D[0:12, 0:8])
# M = 64, both K-major
P = 64
A3 = np.zeros((P, K)); A3[np.arange(K), np.arange(K)] = 1.0
rc, D = run(A3, B, P, Q, K, 0, 0)
print(f"--- M=64 A=I K-major rc={rc}: D[:, 0] ="); print(D[:, 0])
