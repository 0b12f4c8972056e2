"""Fit the tile-plan cost model (w4a8_gemm.cu plan_cost_us) to a quick_bench
tile-plan sweep (profiles/r01_tileplan_sweep_v2.jsonl) and report the regret of
the model's choice against the best measured plan."""
import json, math, sys, collections
import numpy as np
from scipy.optimize import least_squares

SMS = 148
def plan(M, N, K, ntok, split):
    if split == 3:  # 2-CTA pair tiles: 256 channels x 256 tokens, BK = 128, 74 pair slots
        tok_tiles = -(-M // 256)
        pairs = -(-(-(-N // 128)) // 2)
        kbt = -(-K // 128)
        tiles = pairs * tok_tiles
        per = -(-tiles // (SMS // 2))
        return dict(M=M, N=N, K=K, ntok=256, split=3, bk=128, cps=1, grid=2 * (-(-tiles // per)), ucta=per * kbt,
                    kbt=kbt, tiles=tiles, waves=per)
    bk = 256
    cps = 2 if ntok <= 64 else 1
    if split == 4:  # cluster split-K: one tile per cluster of S decode CTAs
        tok_tiles = -(-M // ntok)
        n_tiles = -(-N // 128)
        kbt = -(-K // 256)
        tiles = n_tiles * tok_tiles
        S = next((c for c in (8, 4, 2) if tiles * c <= SMS * 2 and c <= kbt), 1)
        if S == 1:
            return plan(M, N, K, ntok, 1)
        return dict(M=M, N=N, K=K, ntok=ntok, split=4, bk=bk, cps=2, grid=tiles * S, ucta=-(-kbt // S), kbt=kbt,
                    tiles=tiles, waves=1, S=S)
    slots = SMS * cps
    tok_tiles = -(-M // ntok)
    n_tiles = -(-N // 128)
    kbt = -(-(-(-K // 256) * 256) // bk)
    tiles = n_tiles * tok_tiles
    units = tiles * kbt
    if split == 1:
        grid = min(units, slots)
        ucta = -(-units // grid)
        waves = 0
    else:
        per = -(-tiles // slots)
        grid = -(-tiles // per)
        ucta = per * kbt
        waves = per
    return dict(M=M, N=N, K=K, ntok=ntok, split=split, bk=bk, cps=cps, grid=grid, ucta=ucta, kbt=kbt, tiles=tiles,
                waves=waves)

def cost(th, lp):
    T0, Bsm, Btot, cconv, cmma, f0, f1, e0, e1, T0p, Up, c0, c1 = th
    clk = 1900.0
    if lp['split'] == 3:
        epi = e0 + e1 * min(256, lp['M']) / 16.0
        return T0p + lp['ucta'] * Up + lp['waves'] * epi
    bw = min(Bsm * 1e3, Btot * 1e3 / lp['grid'])           # bytes/us per CTA
    wkb = lp['bk'] * 64.0 * (1 + 1 / 32)                   # packed weight bytes per k-block
    mma = (lp['bk'] / 32.0) * (lp['ntok'] / 2.0) / clk * cmma
    conv = lp['bk'] * 128.0 * cconv * 1e-6 * lp['cps']
    u = max(wkb / bw, conv, mma)
    epi = e0 + e1 * min(lp['ntok'], lp['M']) / 16.0
    if lp['split'] == 4:  # no cross-CTA fix-up; cluster launch / DSMEM exchange
        return T0 + c0 + lp['ucta'] * u + epi + c1 * min(lp['ntok'], lp['M']) / 16.0
    if lp['split'] == 1:
        fix = f0 + f1 * min(lp['ntok'], lp['M']) / 16.0
        return T0 + lp['ucta'] * u + fix + epi
    return T0 + lp['ucta'] * u + lp['waves'] * epi

rows = []
for l in (l for f in sys.argv[1:] for l in open(f)):
    if not l.startswith('{'):
        continue
    d = json.loads(l)
    if d['cfg'] is None or d['cfg'].get('split', 1) == 2 or d['scheme'] != 'per-group':
        continue
    k, n = map(int, d['shape'].split('x'))
    rows.append((plan(d['M'], n, k, d['cfg']['ntok'], d['cfg']['split']), d['us']))

def resid(th):
    return np.array([math.log(cost(th, lp)) - math.log(t) for lp, t in rows])

th0 = [2.5, 40.0, 6500.0, 25.0, 1.5, 2.0, 0.2, 1.0, 0.2, 5.0, 0.35, 0.5, 0.1]
r = least_squares(resid, th0, bounds=([0, 1, 100, 0, 0.5, 0, 0, 0, 0, 0, 0.05, -5, -5],
                                      [20, 500, 20000, 500, 10, 50, 10, 20, 10, 30, 2, 10, 10]))
th = r.x
print("theta =", ", ".join("%.4g" % v for v in th))
print("rms log err %.3f" % np.sqrt(np.mean(resid(th) ** 2)))
groups = collections.defaultdict(list)
for lp, t in rows:
    groups[(lp['N'], lp['K'], lp['M'])].append((cost(th, lp), t, lp['ntok'], lp['split']))
tot_best = tot_pick = 0
for key, g in sorted(groups.items()):
    best = min(g, key=lambda x: x[1])
    pick = min(g, key=lambda x: x[0])
    tot_best += best[1]
    tot_pick += pick[1]
    print(key, "best %d%s %.1f  pick %d%s %.1f" % (best[2], 'ws?pc'[best[3]], best[1], pick[2], 'ws?pc'[pick[3]], pick[1]))
print("sum best %.1f  sum picked %.1f  regret %.1f%%" % (tot_best, tot_pick, 100 * (tot_pick / tot_best - 1)))
