"""Phase stamps of the sweep (cluster 0): chain lane 0 and near thread 0, positions 64..319.

    python tools/trace_sweep.py c4 [T] [dirs: fwd|post]
"""
import os
import sys

import numpy as np

os.environ.setdefault("SCRF_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                               "paper_2604_18780_b200", "libscrf_trace.so"))
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18780_b200 as scrf  # noqa: E402
from paper_2604_18780_b200 import _lib  # noqa: E402
from paper_2604_18780_b200 import streaming as S  # noqa: E402
from paper_2604_18780_b200.instances import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
_, params, cum = scrf.equivalence_instance(0, T=T, K=cfg["K"], C=cfg["C"], B=cfg["B"], mode=scrf.CenteringMode.MEAN)
prob = scrf.DeviceProblem.from_host(cum, params)
post = len(sys.argv) > 3 and sys.argv[3] == "post"
run = (lambda: S.device_posterior(prob)) if post else (lambda: S.device_forward(prob))
run()
buf = torch.zeros((1344 + 64, 16), dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.scrf_debug_trace(buf.data_ptr())
run()
lib.scrf_debug_trace(None)
torch.cuda.synchronize()
trall = buf.cpu().numpy().astype(np.float64)
tr = trall[:256]
tl = trall[256:512]
gt = buf.cpu().numpy()[512:].reshape(-1)[: 256 * 4].reshape(256, 4).astype(np.float64)
ch, nr = tr[:, 0:8], tr[:, 8:16]
dd = np.diff(ch[:, 0])
print("chain (median cycles): step", np.median(dd), "mean", dd.mean(), "p10/p50/p90", np.percentile(dd, [10, 50, 90]))
print("  step pattern (first 24):", dd[:24].astype(int).tolist())
names = ["B+lse3", "max+gemv", "publish+arrive"]
for i, n in enumerate(names):
    print(f"  {n:14s} {np.median(ch[:, i + 1] - ch[:, i]):8.0f}")
print("near (median cycles): step", np.median(np.diff(nr[:, 0])))
names = ["sync A", "prep", "ring_lse", "tail+part"]
for i, n in enumerate(names):
    print(f"  {n:14s} {np.median(nr[:, i + 1] - nr[:, i]):8.0f}")
print("near start - chain start (median):", np.median(nr[:, 0] - ch[:, 0]))

if tl[:, 0].any():
    print("tail warp0 (median cycles): step/group", np.median(np.diff(tl[:, 0])))
    seq = [(0, 9, "staging wait"), (9, 1, "source wait"), (1, 4, "e (fp64)"), (4, 5, "re-arm+exact"), (5, 2, "block fma"), (2, 6, "max+ex2"),
           (6, 7, "shfl sums"), (7, 8, "send+stage"), (8, 3, "block complete")]
    for a0, b0, n in seq:
        print(f"  {n:14s} {np.median(tl[:, b0] - tl[:, a0]):8.0f}")
    # near group 0 handles even p; near tr[5..6] = tail wait
    ev = nr[::2]
    print("near tail wait (median):", np.median(ev[:, 6] - ev[:, 5]), " ring write time - tail src arrival")
    # align: tail target u (row u-64) src arrival tl[:,2]; near sends source q at iteration q+4 (tr[7] of row q+4-64)
    ks = 11
    # near row index for iteration p = row p-64; source q sent at iteration q+4; tail target u uses source u-ks
    lat = []
    for r in range(0, 256):
        u = r + 64; q = u - ks; pr = q + 4 - 64
        if 0 <= pr < 256 and nr[pr, 7] > 0 and tl[r, 2] > 0:
            lat.append(tl[r, 2] - nr[pr, 7])
    if lat: print("source send -> tail wakeup (median cycles):", np.median(lat))
    lat = []
    for r in range(0, 256):
        if nr[r, 6] > 0 and tl[r, 3] > 0:
            lat.append(nr[r, 6] - tl[r, 3])
    if lat: print("tail lse done (warp0) -> near wakeup (median):", np.median(lat))

# global-timer latencies (ns): near send source q -> tail sees it; tail sends partial of u -> near receives
kc = 16
lat1 = [gt[r, 1] - gt[r, 0] for r in range(256) if gt[r, 0] > 0 and gt[r, 1] > 0]
lat2 = [gt[r, 3] - gt[r, 2] for r in range(256) if gt[r, 2] > 0 and gt[r, 3] > 0]
lat3 = []  # source q sent -> partial of target q+kc+1+... received (round trip through the tail)
for r in range(256):
    u = r  # target index relative; source u-kc-1
    if r - kc - 1 >= 0 and gt[r - kc - 1, 0] > 0 and gt[r, 3] > 0:
        lat3.append(gt[r, 3] - gt[r - kc - 1, 0])
for n, l in (("src send->tail seen (ns)", lat1), ("partial send->near seen (ns)", lat2), ("source q sent -> partial q+17 received (ns)", lat3)):
    if l: print(f"{n}: median {np.median(l):.0f}  p90 {np.percentile(l, 90):.0f}")
st = [gt[r + 1, 0] - gt[r, 0] for r in range(255) if gt[r, 0] > 0 and gt[r + 1, 0] > 0]
if st: print("near source sends: median interval (ns)", np.median(st))

ax = buf.cpu().numpy()[576:].astype(np.float64)
if ax[:, 0].any():
    print("aux (median cycles): step", np.median(np.diff(ax[:, 0])))
    for a0, b0, n in ((0, 1, "wait+sync A"), (1, 2, "outputs+oq+edge+stage"), (2, 3, "n+bookkeeping")):
        print(f"  {n:22s} {np.median(ax[:, b0] - ax[:, a0]):8.0f}")

g1 = buf.cpu().numpy()[832:].astype(np.float64)
g0 = nr
for name, arr, par in (("near group0 (even p)", g0, 0), ("near group1 (odd p)", g1, 1)):
    rows = arr[par::2] if par == 0 else arr[1::2]
    rows = rows[rows[:, 0] > 0]
    if len(rows) > 2:
        print(name, "iteration (median cycles):", np.median(np.diff(rows[:, 0])))
        for a0, b0, n in ((0, 1, "sync A"), (1, 2, "prep"), (2, 3, "ring_lse"), (3, 5, "pre-tail"), (5, 6, "tail wait"), (6, 4, "merge+part+edge")):
            print(f"  {n:16s} {np.median(rows[:, b0] - rows[:, a0]):8.0f}")

# arrival-side analysis (same SM clock): chainA[p] = chain arrives A(p); nearB[p] = near arrives B(p)
chainA = {}
nearB = {}
base = int(os.environ.get("SCRF_TRACE_FROM", "64"))
for r in range(256):
    p = base + r
    if ch[r, 3] > 0: chainA[p] = ch[r, 3]
    row = nr[r] if (p % 2 == 0) else g1[r]
    if row[4] > 0: nearB[p] = row[4]
Wn, Lc = [], []
for p in range(base + 8, base + 250):
    if p in nearB and (p - 2) in nearB and (p - 4) in chainA:
        Wn.append(nearB[p] - max(nearB[p - 2], chainA[p - 4]))
    if p in chainA and (p - 1) in chainA and p in nearB:
        Lc.append(chainA[p] - max(chainA[p - 1], nearB[p]))
if Wn:
    print("near work per iteration (B(p) - max(B(p-2), A(p-4))): median", np.median(Wn), "p90", np.percentile(Wn, 90))
    print("chain work per step (A(p) - max(A(p-1), B(p))): median", np.median(Lc), "p90", np.percentile(Lc, 90))
    slackA = [nearB[p] - chainA[p - 4] for p in range(base + 8, base + 250) if p in nearB and (p - 4) in chainA]
    print("B(p) - A(p-4): median", np.median(slackA))
    lat = [chainA[p] - nearB[p] for p in range(base + 8, base + 250) if p in nearB and p in chainA]
    print("A(p) - B(p): median", np.median(lat))

# globaltimer timeline (ns) of cluster 0, 8 slots per position
G = buf.cpu().numpy()[1088:].reshape(-1)[: 256 * 8].reshape(256, 8).astype(np.float64)
names = ["src sent", "tail saw", "tail sent", "near got", "chain B", "chain A", "near A-4", "edge done"]
def col(i):
    return G[:, i]
def med(xs):
    xs = [v for v in xs if v == v]
    return (np.mean(xs), np.percentile(xs, 90)) if xs else (float("nan"), float("nan"))
print("\nglobaltimer (ns) means [p90] (256 ns ticks):")
def pairs(desc, fa, fb):
    v = []
    for r in range(256):
        a0, b0 = fa(r), fb(r)
        if a0 is not None and b0 is not None and a0 > 0 and b0 > 0:
            v.append(b0 - a0)
    m = med(v)
    print(f"  {desc:52s} {m[0]:8.0f} [{m[1]:8.0f}]")
def g(r, i):
    return G[r, i] if 0 <= r < 256 else None
pairs("chain A(p) -> A(p+1) (step)", lambda r: g(r, 5), lambda r: g(r + 1, 5))
pairs("chain B(p) -> A(p) (chain work)", lambda r: g(r, 4), lambda r: g(r, 5))
pairs("chain A(p-1) -> B(p) (wait for B)", lambda r: g(r - 1, 5), lambda r: g(r, 4))
pairs("chain A(p-4) -> near passes A(p-4)", lambda r: g(r - 4, 5), lambda r: g(r, 6))
pairs("near passes A(p-4) -> near got tail(p)", lambda r: g(r, 6), lambda r: g(r, 3))
pairs("near got tail(p) -> chain B(p)", lambda r: g(r, 3), lambda r: g(r, 4))
pairs("chain A(q) -> src sent q", lambda r: g(r, 5), lambda r: g(r, 0))
pairs("src sent q -> tail saw q", lambda r: g(r, 0), lambda r: g(r, 1))
pairs("tail saw q=u-14 -> tail sent u (u=group first)", lambda r: g(r - 14, 1), lambda r: g(r, 2))
pairs("tail sent u -> near got u", lambda r: g(r, 2), lambda r: g(r, 3))
pairs("tail saw q -> tail saw q+4 (group period)", lambda r: g(r, 1), lambda r: g(r + 4, 1))
pairs("src sent q+3 -> tail saw q+3 (q = group's sb)", lambda r: g(r, 0) if (base + r - 17) % 4 == 3 else None, lambda r: g(r, 1))
pairs("tail saw sb+3 -> tail sent u (u = sb+17 .. )", lambda r: g(r - 14, 1) if (base + r - 17) % 4 == 0 else None, lambda r: g(r, 2))
pairs("chain A(q) (q%4==0) -> edge done", lambda r: g(r, 5) if (base + r) % 4 == 0 else None, lambda r: g(r, 7))
print("  per residue p%4 of chain step A(p-1)->A(p):", [float(np.mean([G[r, 5] - G[r - 1, 5] for r in range(1, 256) if (base + r) % 4 == k and G[r, 5] > 0 and G[r - 1, 5] > 0])) for k in range(4)])
print("  per residue p%4 of near got tail(p) - near passes A(p-4):", [float(np.mean([G[r, 3] - G[r, 6] for r in range(0, 256) if (base + r) % 4 == k and G[r, 3] > 0 and G[r, 6] > 0])) for k in range(4)])

# head-clock round trip: source sb+3 sent (src warp) -> partial of target sb+17 received (near)
srcs = buf.cpu().numpy()[576:832, 0].astype(np.float64)
nearA = {}
rt, win = [], []
for r in range(256):
    p = base + r
    sb = p - 17
    if (sb % 4) == 0 and 0 <= r - 14 < 256 and srcs[r - 14] > 0:
        row = nr[r] if (p % 2 == 0) else g1[r] if r < len(g1) else None
        if row is not None and row[6] > 0:
            rt.append(row[6] - srcs[r - 14])
            if (p - 4) in chainA:
                win.append(chainA[p - 4] - srcs[r - 14])
if rt:
    print("head clock: source sb+3 sent -> near got partial of sb+17: mean", np.mean(rt), "median", np.median(rt))
    print("head clock: source sb+3 sent -> chain arrives A(sb+13):   mean", np.mean(win))

ts = buf.cpu().numpy()[1216:].reshape(-1)[: 16 * 16 * 4].reshape(16 * 16, 4)
print("tail warps (cluster 0, targets >= 1000): tail, warp, source-wait %, slow groups")
for i in range(16 * 16):
    if ts[i, 1] > 0:
        print(f"  tail {i // 16 + 1} warp {i % 16:2d}: wait {100.0 * ts[i, 0] / ts[i, 1]:5.1f}%  slow {ts[i, 2]}")

cb = buf.cpu().numpy()[1280:].reshape(-1).astype(np.float64)
snd, ech, rcv = cb[0:64], cb[64:128], cb[128:192]
if (snd > 0).all() and (rcv > 0).all():
    rtt = rcv - snd
    off = ech - (snd + rcv) / 2  # tail clock - head clock
    print(f"gt calibration: head<->tail1 global-flag rtt mean {rtt.mean():.0f} ns; offset (tail - head) mean {off.mean():.0f} ns")

tw = buf.cpu().numpy()[1312:].reshape(-1)[:512].reshape(256, 2).astype(np.float64)
off_th = off.mean() if (snd > 0).all() and (rcv > 0).all() else 0.0
d_start, d_saw, ready = [], [], []
for r in range(256):
    if tw[r, 0] > 0 and G[r, 0] > 0 and G[r, 1] > 0:
        d_start.append(tw[r, 0] - off_th - G[r, 0])  # tail wait start - head sent (head clock)
        d_saw.append(G[r, 1] - off_th - G[r, 0])
        ready.append(tw[r, 1] == 1)
if d_start:
    print(f"tail group wait for source q=sb+3: start - sent {np.mean(d_start):.0f} ns, saw - sent {np.mean(d_saw):.0f} ns, "
          f"already complete at start {100.0 * np.mean(ready):.0f}%")

ss = buf.cpu().numpy()[1344:].reshape(-1)[: 256 * 4].reshape(256, 4).astype(np.float64)
ok = ss[:, 0] > 0
if ok.sum() > 4:
    it = np.diff(ss[ok, 0])
    print("source warp (median cycles): iteration", np.median(it), "| wait at A", np.median(ss[ok, 1] - ss[ok, 0]),
          "| A -> ring written", np.median(ss[ok, 2] - ss[ok, 1]), "| ring -> sends issued", np.median(ss[ok, 3] - ss[ok, 2]),
          "| sends -> next loop top", np.median(ss[1:, 0][ok[1:]] - ss[:-1, 3][ok[1:]]))
