"""W4 kernel per-stage timeline of one CTA (RTNQ_WGEMM_DEBUG = 512 | cta << 16), profiling build:
RTNQ_LIB=paper_2505_15909_b200/librtnq_b200_dbg.so CTA=5 B=16 python scratch/i4tl.py"""
import os, sys, ctypes, torch, numpy as np
sys.path.insert(0, os.getcwd())
cta = int(os.environ.get("CTA", "5"))
os.environ["RTNQ_WGEMM_DEBUG"] = str(512 | (cta << 16) | int(os.environ.get("DBG", "0")))
import paper_2505_15909_b200 as rq
L = rq.lib()
B = int(os.environ.get("B", "16"))
n, k = 28672, 4096
w = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
q = rq.quantize_pack(w, 4, 128)
x = torch.empty(B, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
ws = rq.Workspace(device="cuda")
for _ in range(3):
    rq.linear(x, q, workspace=ws, check=False)
torch.cuda.synchronize()
buf = np.zeros(64 * 16, np.int64)
L.rtnq_i4_timeline_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
T = buf.reshape(64, 16)
if os.environ.get("PROLOGUE"):
    print("prologue: mbar_init", T[63][13], "alloc", T[63][14], "syncthreads", T[63][15], "own planes: start", T[62][5], "produced", T[62][6], "tp: enter/scan/exp/split/bar/released", list(T[61][:6]), "planes producer loop", T[62][13], "codes producer loop", T[62][14], "loop body start", T[62][10], "after expect", T[62][11], "after codes bulk", T[62][12], "first codes TMA", T[0][0], "stage0 exp start", T[0][2], "mma start", T[0][4])
    sys.exit(0)
t = T
ev = ["tmaC", "mmaI", "expS", "expE", "mmaS", "mmaE", "epiS", "epiE"]
if os.environ.get("FULL"):
    names = ["tmaC", "mmaI", "expS", "expE", "mmaS", "mmaE", "epiS", "epiE", "mFull", "mAful", "", "xFull", "xAemp"]
    print("stage " + " ".join(f"{e:>6s}" for e in names if e))
    for i in range(64):
        if T[i].max() == 0:
            break
        print(f"{i:5d} " + " ".join(f"{T[i][j]:6d}" for j in range(13) if names[j]))
    sys.exit(0)
t = T[:, :8]
print("stage " + " ".join(f"{e:>7s}" for e in ev) + "   exp  mma issue commit  epi  epi-gap mma-gap")
import statistics
rows = [i for i in range(64) if t[i].max() > 0]
if os.environ.get("SUMMARY"):
    st = [t[i][4] - t[i - 1][4] for i in rows[6:-2]]
    print(f"DBG={os.environ.get('DBG','0')} B={B}: stage period {statistics.median(st):.0f}, mma issue {statistics.median([t[i][1]-t[i][4] for i in rows[6:-2]]):.0f}, commit {statistics.median([t[i][5]-t[i][1] for i in rows[6:-2]]):.0f}, exp {statistics.median([t[i][3]-t[i][2] for i in rows[6:-2]]):.0f}, epi {statistics.median([t[i][7]-t[i][6] for i in rows[6:-2]]):.0f}, mma-gap {statistics.median([t[i][4]-t[i-1][5] for i in rows[6:-2]]):.0f}")
    t = T
    print("  mma: wait full", statistics.median([t[i][8]-t[i-1][5] for i in rows[6:-2]]),
          "then afull", statistics.median([t[i][9]-t[i][8] for i in rows[6:-2]]), "then tfree", statistics.median([t[i][4]-t[i][9] for i in rows[6:-2]]),
          "| exp: wait full", statistics.median([t[i][11]-t[i-1][3] for i in rows[6:-2]]), "then aempty", statistics.median([t[i][12]-t[i][11] for i in rows[6:-2]]),
          "then tfree", statistics.median([t[i][2]-t[i][12] for i in rows[6:-2]]))
    sys.exit(0)
for i in range(64):
    if t[i].max() == 0:
        break
    prev = t[i - 1][7] if i else 0
    print(f"{i:5d} " + " ".join(f"{v:7d}" for v in t[i]) +
          f" {t[i][3] - t[i][2]:5d} {t[i][5] - t[i][4]:4d} {t[i][1] - t[i][4]:5d} {t[i][5] - t[i][1]:6d} {t[i][7] - t[i][6]:4d} {t[i][6] - prev:5d} {t[i][4] - (t[i - 1][5] if i else 0):7d}")
