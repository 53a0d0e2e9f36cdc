import sys, numpy as np
t = np.fromfile(sys.argv[1], dtype=np.uint64)[:8 * 4096].reshape(8, 4096).astype(np.int64)
names = ["codeIssue", "xIssue", "mma_afull", "mma_xfull", "dq_cfull", "dq_computed", "dq_aempty", "dq_st"]
n = [int((t[s] > 0).sum()) for s in range(8)]
t0 = min(int(t[s][t[s] > 0].min()) for s in range(8) if n[s])
print("events per slot", dict(zip(names, n)))
N = min(n[2], n[4], 40)
print(" c  " + " ".join(f"{x:>11}" for x in names))
for c in list(range(0, min(N, 24))) + list(range(max(0, n[2] - 8), n[2])):
    print(f"{c:3d} " + " ".join(f"{(t[s][c]-t0) if t[s][c] else -1:>11d}" for s in range(8)))
tot = t[2][n[2]-1] - t0
print("total cycles", tot, "chunks", n[2], "cycles/chunk", tot / max(1, n[2]))
d = lambda a, b: np.median((t[b][:N] - t[a][:N]))
print("median cfull->computed", d(4, 5), " computed->aempty", d(5, 6), " aempty->st", d(6, 7))
print("median gaps MMA afull: ", np.median(np.diff(t[2][:n[2]])), " code issue gaps", np.median(np.diff(t[0][:n[0]])), " x issue gaps", np.median(np.diff(t[1][:n[1]])))
