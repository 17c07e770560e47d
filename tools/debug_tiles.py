"""Debug aid: qgemm (packed path) vs the one-thread-per-output qgemm_naive in
exact-integer mode (bitwise); reports mismatching 64x64 tiles and
their ids in the grouped raster (to tell data-parallel from stream-K tiles).

    python tools/debug_tiles.py [repeats] [M N K]
"""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg

def run(M, N, K, ops="NH", beta=1.0, same=False):
    g = torch.Generator(device="cuda").manual_seed(1)
    ar, ac = (M, K) if ops[0] == "N" else (K, M)
    br, bc = (K, N) if ops[1] == "N" else (N, K)
    A = torch.randint(-8, 9, (ac, ar, 4), generator=g, device="cuda").double()
    B = A if same else torch.randint(-8, 9, (bc, br, 4), generator=g, device="cuda").double()
    C = torch.randint(-8, 9, (N, M, 4), generator=g, device="cuda").double()
    C2 = C.clone()
    old = qg.set_path_policy(qg.PATH_PACKED)
    qg.qgemm(ops[0], ops[1], 1.0, A, B, beta, C, M=M, N=N, K=K)
    qg.set_path_policy(old)
    qg.qgemm_naive(ops[0], ops[1], 1.0, A, B, beta, C2, M=M, N=N, K=K)
    torch.cuda.synchronize()
    d = (C - C2).abs().amax(dim=2)  # (N, M)
    bad = (d > 0).nonzero()
    if bad.numel() == 0:
        print(M, N, K, ops, "OK", flush=True); return
    tiles = sorted(set((int(r) // 64, int(c) // 64) for c, r in bad[:100000].tolist()))
    MT, NT = (M + 63) // 64, (N + 63) // 64
    # tile id in the grouped raster (groups of 8 M-tiles)
    def tid(mt, nt):
        g = mt // 8; gsz = min(8, MT - g * 8)
        return g * 8 * NT + nt * gsz + (mt - g * 8)
    ids = sorted(tid(a, b) for a, b in tiles)
    print(M, N, K, ops, "BAD quats", bad.shape[0], "tiles", len(tiles), tiles[:6], "ids", ids[:12],
          "of", MT * NT, "max", float(d.max()), flush=True)

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
shape = tuple(int(x) for x in sys.argv[2:5]) if len(sys.argv) >= 5 else (32768, 32768, 256)
for _ in range(reps):
    run(*shape, same=shape[0] == shape[1])
