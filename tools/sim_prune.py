"""CPU model of the sweeps' box pruning on one C2 chunk (design aid, not a test).

For a given ordering it reports, per pass, the fraction of (warp x sub-tile)
blocks evaluated and, inside evaluated blocks, the fraction of (ref, cand)
pairs that need the full distance (A <= eps for counts, partial <= eps for
kNN) and the probability that a candidate needs it for ANY ref of the warp.
"""
import sys, os
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import oracle
from paper_1401_4068_b200 import workloads

def morton(pts, cols, bits):
    q = []
    for c in cols:
        v = pts[:, c]; lo, hi = v.min(), v.max()
        q.append(np.clip(((v - lo) / (hi - lo) * (2**bits - 1)), 0, 2**bits - 1).astype(np.uint64))
    key = np.zeros(len(pts), np.uint64)
    for b in range(bits - 1, -1, -1):
        for qi in q:
            key = (key << np.uint64(1)) | ((qi >> np.uint64(b)) & np.uint64(1))
    return np.argsort(key, kind="stable")

def boxes(p, g):
    n = len(p) // g * g
    b = p[:n].reshape(-1, g, p.shape[1])
    return b.min(1), b.max(1)

def sim(pts, eps, order, fcols, name, wsize=128, sub=32, ref_lanes=32):
    p = pts[order]; e = eps[order]
    n = len(p) // wsize * wsize
    p, e = p[:n], e[:n]
    wlo, whi = boxes(p, wsize); slo, shi = boxes(p, sub)
    tot_blocks = 0; ev_blocks = 0; pairs = 0; need = 0; cand_any = 0; cands = 0; lane_any = 0; lanes = 0; grp_any = 0; grps = 0
    for w in range(len(wlo)):
        bound = e[w*wsize:(w+1)*wsize].max()
        bd = np.maximum(slo[:, fcols] - whi[w, fcols], wlo[w, fcols] - shi[:, fcols]).max(1)
        sel = np.nonzero(bd <= bound)[0]
        tot_blocks += len(slo); ev_blocks += len(sel)
        refs = p[w*wsize:(w+1)*wsize][:, fcols]; re = e[w*wsize:(w+1)*wsize]
        for s in sel:
            c = p[s*sub:(s+1)*sub][:, fcols]
            A = np.abs(refs[:, None, :] - c[None, :, :]).max(2)   # [128, 32]
            m = A <= re[:, None]
            pairs += m.size; need += m.sum()
            cand_any += m.any(0).sum(); cands += m.shape[1]
            # lane = 4 refs r*32+lane
            lm = m.reshape(4, 32, -1).any(0)   # [32 lanes, 32 cands]
            lane_any += lm.sum(); lanes += lm.size
            gm = m.reshape(4, 32, -1).any(1)   # [4 groups, 32 cands]
            grp_any += gm.sum(); grps += gm.size
    print(f"{name}: evaluated blocks {ev_blocks/tot_blocks:.4f}; pairs needing full {need/pairs:.4f}; "
          f"P(any ref of warp needs cand) {cand_any/cands:.4f}; P(32-group) {grp_any/grps:.4f}; P(lane needs) {lane_any/lanes:.4f}")

def main():
    wl = workloads.CONFIGS["C2"]
    x, y = wl.ensembles()
    joint = oracle.assemble(x, y, wl.spec, wl.spec, 1, wl.window)
    w = wl.window[1] - wl.window[0] + 1
    perm = oracle.draw_permutation(x.shape[0], np.random.SeedSequence((0, 0)))
    sur = oracle.permuted_joint(joint, perm, w, wl.spec[0])
    margs = oracle.te_margs(3, 3)
    for tag, pts in (("orig", joint), ("surr", sur)):
        eps, cnt = oracle.search(pts, margs, 4)
        print(tag, "counts mean", [float(np.mean(c)) for c in cnt])
        yp = [1, 2, 3]; allc = list(range(7))
        o_y = morton(pts, yp, 10)
        o_all = morton(pts, allc, 4)
        sim(pts, eps, o_y, yp, f"{tag} count/ypast-order")


main()
