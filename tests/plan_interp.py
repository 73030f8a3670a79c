"""Host replay of libtt's kernel index arithmetic from a plan's JSON
description (tt_plan_describe), used by the CPU tests to check the planner's
geometry against the oracle without a GPU.  Test infrastructure only."""
import numpy as np


def interpret_tile_plan(j, words, out=None):
    """Replay the tile kernel's index arithmetic (kernels.cu) for plan JSON j:
    Algorithm-1 decode of the tile base, Eq. (4) input-order minor offsets,
    staging positions, Eq. (5)/(6) output-order offsets, ragged-chunk masks.
    ``out``: write into this buffer (strided plans) instead of a new dense
    array; every touched position must be written exactly once."""
    t = j["tile"]
    V, a = t["V"], len(t["ext"])
    ext, cin, order = t["ext"], t["cin"], t["out_order"]
    sin, sout = t["sin"], t["sout"]
    sm = t["sm"]
    st, sl, sc, se = t["split_tile"], t["split_lane"], t["split_chunk"], t["split_ext"]
    tails = [se[s] - (-(-se[s] // sc[s]) - 1) * sc[s] for s in range(len(st))]
    gC, gD, gSi, gSo = t["grid_c"], t["grid_d"], t["grid_sin"], t["grid_sout"]
    vol = int(np.prod(j["dims"]))
    if out is None:
        out = np.zeros(vol, dtype=words.dtype)
    written = np.zeros(out.size, dtype=np.int64)
    # per-slot tables
    gin, pin, cin_s = [], [], []
    for k in range(V):
        rem, off, cs = k, 0, [0, 0]
        for i in range(a):
            c = rem % ext[i]
            rem //= ext[i]
            off += c * sin[i]
            for s in range(len(st)):
                if st[s] == i:
                    cs[s] = c
        gin.append(off)
        rem, sp = k, 0
        for i in range(a):
            sp += (rem % ext[i]) * sm[i]
            rem //= ext[i]
        pin.append(sp)
        cin_s.append(cs)
    assert len(set(pin)) == V and max(pin) < t["sbuf"]
    gout, psh, cout_s = [], [], []
    for k in range(V):
        rem, off, sh, cs = k, 0, 0, [0, 0]
        for ti in order:
            c = rem % ext[ti]
            rem //= ext[ti]
            off += c * sout[ti]
            sh += c * sm[ti]
            for s in range(len(st)):
                if st[s] == ti:
                    cs[s] = c
        gout.append(off)
        psh.append(sh)
        cout_s.append(cs)
    if "sd" in t:
        return _interpret_sd(j, t, words, tails, out)
    for tile in range(t["nTiles"]):
        q = [(tile // gC[g]) % gD[g] for g in range(len(gC))]
        ib = sum(q[g] * gSi[g] for g in range(len(gC)))
        ob = sum(q[g] * gSo[g] for g in range(len(gC)))
        ragged = [q[sl[s]] == gD[sl[s]] - 1 for s in range(len(st))]
        smem = {}
        for k in range(V):
            if all((not ragged[s]) or cin_s[k][s] < tails[s] for s in range(len(st))):
                smem[pin[k]] = words[ib + gin[k]]
        for k in range(V):
            if all((not ragged[s]) or cout_s[k][s] < tails[s] for s in range(len(st))):
                out[ob + gout[k]] = smem[psh[k]]
                written[ob + gout[k]] += 1
    assert written.max() <= 1 and written.sum() == vol, "tile decomposition must cover every output once"
    return out


def _sd_phase(j, t, ph, tails):
    """Per ragged state need = 0..3, the (global offset, staging offset)
    pairs one phase of tile_sd_kernel touches: thread u = tid + q*threads
    decodes the phase's thread space (slot dim replaced by its chunk index),
    slot r adds r * stride along the slot dim, valid slots are r < cnt."""
    sd = t["sd"]
    ext, sm = t["ext"], t["sm"]
    stride = t["sin"] if ph == 0 else t["sout"]
    order = list(range(len(ext))) if ph == 0 else t["out_order"]
    sl, R, C, U, Q = sd["slot"][ph], sd["R"][ph], sd["C"][ph], sd["U"][ph], sd["Q"][ph]
    assert R <= sd["r"] and Q <= sd["q"] and U <= j["threads"] * Q
    st = t["split_tile"]
    lists = [[] for _ in range(4)]
    for tid in range(j["threads"]):
        for qq in range(Q):
            u = tid + qq * j["threads"]
            if u >= U:
                continue
            rem, off, sp, xs, bad = u, 0, 0, 0, 0
            for ti in order:
                e = C if ti == sl else ext[ti]
                c = rem % e
                rem //= e
                if ti == sl:
                    c *= R
                    xs = c
                else:
                    for s in range(len(st)):
                        if st[s] == ti and c >= tails[s]:
                            bad |= 1 << s
                off += c * stride[ti]
                sp += c * sm[ti]
            for n in range(4):
                if bad & n:
                    continue
                lim = ext[sl]
                for s in range(len(st)):
                    if st[s] == sl and n & (1 << s):
                        lim = tails[s]
                cnt = min(max(lim - xs, 0), R)
                for r in range(cnt):
                    lists[n].append((off + r * stride[sl], sp + r * sm[sl]))
    return lists


def _interpret_sd(j, t, words, tails, out=None):
    st, sl = t["split_tile"], t["split_lane"]
    gC, gD, gSi, gSo = t["grid_c"], t["grid_d"], t["grid_sin"], t["grid_sout"]
    vol = int(np.prod(j["dims"]))
    if out is None:
        out = np.zeros(vol, dtype=words.dtype)
    written = np.zeros(out.size, dtype=np.int64)
    load, store = _sd_phase(j, t, 0, tails), _sd_phase(j, t, 1, tails)
    for n in range(4):
        pos = [p for _, p in load[n]]
        assert len(set(pos)) == len(pos) and (not pos or max(pos) < t["sbuf"])
    for tile in range(t["nTiles"]):
        q = [(tile // gC[g]) % gD[g] for g in range(len(gC))]
        ib = sum(q[g] * gSi[g] for g in range(len(gC)))
        ob = sum(q[g] * gSo[g] for g in range(len(gC)))
        need = sum(1 << s for s in range(len(st)) if q[sl[s]] == gD[sl[s]] - 1
                   and tails[s] != t["split_chunk"][s])
        smem = {p: words[ib + g] for g, p in load[need]}
        for g, p in store[need]:
            out[ob + g] = smem[p]
            written[ob + g] += 1
    assert written.max() <= 1 and written.sum() == vol, "slot-dim tiles must cover every output once"
    return out


def interpret_tiled2d_plan(j, words, out=None):
    """Replay the 2-D kernel's tile geometry: grid decode (Algorithm 1),
    ragged limits, and out[ob + a*sOutA + b] = in[ib + b*sInB + a]."""
    t = j["tiled2d"]
    TA, TB = t["TA"], t["TB"]
    gC, gD, gSi, gSo = t["grid_c"], t["grid_d"], t["grid_sin"], t["grid_sout"]
    vol = int(np.prod(j["dims"]))
    if out is None:
        out = np.zeros(vol, dtype=words.dtype)
    written = np.zeros(out.size, dtype=np.int64)
    for tile in range(t["nTiles"]):
        q = [(tile // gC[g]) % gD[g] for g in range(len(gC))]
        ib = sum(q[g] * gSi[g] for g in range(len(gC)))
        ob = sum(q[g] * gSo[g] for g in range(len(gC)))
        la, lb = t["lanes"]
        limA = t["tails"][0] if q[la] == gD[la] - 1 else TA
        limB = t["tails"][1] if q[lb] == gD[lb] - 1 else TB
        a = np.arange(limA)[:, None]
        b = np.arange(limB)[None, :]
        dst = (ob + a * t["sOutA"] + b).ravel()
        out[dst] = words[(ib + b * t["sInB"] + a).ravel()]
        written[dst] += 1
    assert written.max() <= 1 and written.sum() == vol, "2-D tiles must cover every output once"
    return out



def interpret_rowcopy_plan(j, words):
    """Replay the row-copy kernel: output row r = contiguous input row at
    sum_j digit_j(r) * row_sin[j]."""
    t = j["rowcopy"]
    n, full, seg, tail, nseg = t["nRows"], t["row_full"], t["seg"], t["seg_tail"], t["nseg"]
    out = np.zeros(full * (n // nseg), dtype=words.dtype)
    for r in range(n):
        base = sum(((r // c) % d) * s for c, d, s in zip(t["row_c"], t["row_d"], t["row_sin"]))
        k = r % nseg                      # segment of the row (digit 0 when segmented)
        L = tail if (nseg > 1 and k == nseg - 1) else seg
        o = (r // nseg) * full + k * seg
        out[o:o + L] = words[base:base + L]
    return out


def interpret_plan(j, words):
    """Output of a (non-sharded) plan description applied to ``words``.
    A widened plan (elem_size = widen x the caller's element) is replayed on
    the same bytes viewed as wider opaque words."""
    E = j["word_size"]
    orig = words.dtype
    if words.dtype.itemsize != E:
        words = np.ascontiguousarray(words).view(np.dtype(f"V{E}"))
    if j["kernel"] == "copy":
        out = np.array(words, copy=True)
    else:
        fj = dict(j)
        fj["dims"] = j["fused"]["dims"]
        if j["kernel"] == "tiled2d":
            out = interpret_tiled2d_plan(fj, words)
        elif j["kernel"] == "rowcopy":
            out = interpret_rowcopy_plan(fj, words)
        else:
            out = interpret_tile_plan(fj, words)
    return out.view(orig)
