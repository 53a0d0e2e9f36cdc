import sys, numpy as np
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(8, 4096).astype(np.int64)
n2 = int((t[2] > 0).sum())
t0 = t[t > 0].min()
print("MMA chunks", n2, "cycles/chunk", (t[2][n2-1] - t[2][1]) / max(1, n2 - 2))
for g in range(4):
    cf = t[4][g*1024:(g+1)*1024]; ae = t[5][g*1024:(g+1)*1024]; af = t[6][g*1024:(g+1)*1024]
    n = int((cf > 0).sum())
    if n < 3: continue
    print(f"grp{g}: n={n} cfull->aempty {np.median(ae[1:n]-cf[1:n]):.0f}  aempty->afull(st+wait) {np.median(af[1:n]-ae[1:n]):.0f}  afull->next cfull {np.median(cf[2:n]-af[1:n-1]):.0f}  period {np.median(np.diff(cf[1:n])):.0f}")
