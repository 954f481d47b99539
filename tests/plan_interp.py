"""Test-only NumPy interpreter of native plan ops (include/atamul_b200.h).

Executes a planner's op list on host arrays with the documented semantics,
so planner logic (windows, signs, truncation, grouping) is checked on the CPU
without a GPU.  Never used by the product path.
"""
import numpy as np

OP_GEMM, OP_SYRK, OP_COMBO, OP_UPDATE, OP_FILL, OP_COMBO4, OP_POSTADD7, OP_ROUND = 0, 1, 2, 3, 4, 5, 6, 7


def _win(bases, r, write=False):
    base = bases[int(r["base"])]
    rows, cols, off, ld = int(r["rows"]), int(r["cols"]), int(r["off"]), int(r["ld"])
    if rows == 0 or cols == 0:
        return None
    flat = base.reshape(-1)
    assert off >= 0 and off + (rows - 1) * ld + cols <= flat.size, "window out of bounds"
    return np.lib.stride_tricks.as_strided(flat[off:], shape=(rows, cols),
                                           strides=(ld * flat.itemsize, flat.itemsize),
                                           writeable=write)


def _operand(bases, refs, count, m, width, dtype):
    out = np.zeros((m, width), dtype=dtype)
    for j in range(count):
        w = _win(bases, refs[j])
        if w is None:
            continue
        r, c = min(w.shape[0], m), min(w.shape[1], width)
        out[:r, :c] += float(refs[j]["sign"]) * w[:r, :c]
    return out


def run(ops, A, C, alpha=1.0, WS=None, B=None):
    dtype = C.dtype
    bases = {0: A, 1: C, 2: WS if WS is not None else np.zeros(1, dtype), 3: B if B is not None else A}
    for op in ops:
        t = int(op["type"])
        if t in (OP_GEMM, OP_SYRK):
            m, n, k = int(op["m"]), int(op["n"]), int(op["k"])
            S = _operand(bases, op["s"], int(op["ns"]), m, n, dtype)
            T = S if t == OP_SYRK else _operand(bases, op["t"], int(op["nt"]), m, k, dtype)
            P = S.T @ T
            for j in range(int(op["nd"])):
                d = op["d"][j]
                w = _win(bases, d, write=True)
                v = alpha * float(d["sign"]) * P[:w.shape[0], :w.shape[1]]
                if t == OP_SYRK:
                    mask = np.tril(np.ones(w.shape, dtype=bool))
                    if int(op["accumulate"]):
                        w[mask] += v[mask]
                    else:
                        w[mask] = v[mask]
                else:
                    if int(op["accumulate"]):
                        w += v
                    else:
                        w[...] = v
        elif t == OP_COMBO:
            d = _win(bases, op["d"][0], write=True)
            d[...] = _operand(bases, op["s"], int(op["ns"]), d.shape[0], d.shape[1], dtype)
        elif t == OP_UPDATE:
            src = _win(bases, op["s"][0])
            for j in range(int(op["nd"])):
                w = _win(bases, op["d"][j], write=True)
                w += float(op["d"][j]["sign"]) * src[:w.shape[0], :w.shape[1]]
        elif t == OP_FILL:
            _win(bases, op["d"][0], write=True)[...] = 0
        elif t == OP_ROUND and int(op["accumulate"]) == 2:
            pass          # L2 rounding ring: the product kernel rounds its operand loads
        elif t == OP_ROUND:   # round-to-nearest (ties away) to TF32, fp32 storage
            src = _win(bases, op["s"][0]).astype(np.float32)
            bits = src.view(np.uint32).astype(np.uint64)
            bits = ((bits + 0x1000) & ~np.uint64(0x1FFF)).astype(np.uint32)
            _win(bases, op["d"][0], write=True)[...] = bits.view(np.float32)
        elif t == OP_POSTADD7:
            kids = [op["s"][q] for q in range(4)] + [op["t"][q] for q in range(3)]
            wins = [_win(bases, r) for r in kids]
            R = max((w.shape[0] for w in wins if w is not None), default=0)
            Cc = max((w.shape[1] for w in wins if w is not None), default=0)
            P = []
            for w in wins:
                z = np.zeros((R, Cc), dtype=dtype)
                if w is not None:
                    z[:w.shape[0], :w.shape[1]] = w
                P.append(z)
            Q = [P[0] + P[3] - P[4] + P[6], P[2] + P[4], P[1] + P[3], P[0] - P[1] + P[2] + P[5]]
            for j in range(4):
                d = _win(bases, op["d"][j], write=True)
                if d is None:
                    continue
                v = float(op["d"][j]["sign"]) * Q[j][:d.shape[0], :d.shape[1]]
                if int(op["accumulate"]):
                    d += v
                else:
                    d[...] = v
        elif t == OP_COMBO4:
            srcs = [_win(bases, op["s"][q]) for q in range(int(op["ns"]))]
            for j in range(int(op["nd"])):
                d = _win(bases, op["d"][j], write=True)
                code = int(op["d"][j]["region"])
                acc = np.zeros(d.shape, dtype=dtype)
                for q, w in enumerate(srcs):
                    cq = (code >> (2 * q)) & 3
                    if cq == 0 or w is None:
                        continue
                    r, c = min(w.shape[0], d.shape[0]), min(w.shape[1], d.shape[1])
                    acc[:r, :c] += (1.0 if cq == 1 else -1.0) * w[:r, :c]
                if int(op["accumulate"]):   # lower-triangular outputs
                    mask = np.tril(np.ones(d.shape, dtype=bool))
                    d[mask] = acc[mask]
                else:
                    d[...] = acc
        else:
            raise ValueError(t)
    return C
