"""Dev probe: pinned host <-> device copy rates, one large copy vs the e2e step's per-layer pieces."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench


def main():
    dev = torch.device("cuda", 0)
    local = bench.gpu_local_cpus(dev)
    if local:
        os.sched_setaffinity(0, local)
    MB = 1 << 20
    # e2e per-layer pieces (cfg 2): prefill q 16 MiB, k 4, v 4; decode q 0.5, k/v 128 KiB
    pieces = [16 * MB, 4 * MB, 4 * MB, MB // 2, MB // 8, MB // 8] * 32
    tot = sum(pieces)
    h = torch.empty(tot, dtype=torch.uint8).pin_memory()
    d = torch.empty(tot, dtype=torch.uint8, device=dev)
    ho = torch.empty(tot * 2 // 3, dtype=torch.uint8).pin_memory()
    do = torch.empty(tot * 2 // 3, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) / reps

    def one():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)

    def many():
        with torch.cuda.stream(s1):
            o = 0
            for p in pieces:
                d[o:o + p].copy_(h[o:o + p], non_blocking=True)
                o += p

    def per_layer():
        with torch.cuda.stream(s1):
            n = tot // 32
            for l in range(32):
                d[l * n:(l + 1) * n].copy_(h[l * n:(l + 1) * n], non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)

    def both():
        one(); d2h()

    opieces = [16 * MB, MB // 2] * 32

    def d2h_pieces():
        with torch.cuda.stream(s2):
            o = 0
            for p in opieces:
                ho[o:o + p].copy_(do[o:o + p], non_blocking=True)
                o += p

    def both_pieces():
        many(); d2h_pieces()

    def both_layer():
        per_layer()
        with torch.cuda.stream(s2):
            n = sum(opieces) // 32
            for l in range(32):
                ho[l * n:(l + 1) * n].copy_(do[l * n:(l + 1) * n], non_blocking=True)

    def both_interleaved():
        # the e2e pattern: per layer, H2D pieces then the D2H of that layer after an event
        evs = [torch.cuda.Event() for _ in range(32)]
        with torch.cuda.stream(s1):
            o = 0
            for l in range(32):
                for p in pieces[6 * l:6 * l + 6]:
                    d[o:o + p].copy_(h[o:o + p], non_blocking=True)
                    o += p
                evs[l].record(s1)
        with torch.cuda.stream(s2):
            o = 0
            for l in range(32):
                s2.wait_event(evs[l])
                for p in opieces[2 * l:2 * l + 2]:
                    ho[o:o + p].copy_(do[o:o + p], non_blocking=True)
                    o += p

    for name, fn, nb in (("h2d one", one, tot), ("h2d pieces", many, tot), ("h2d per layer", per_layer, tot),
                         ("d2h one", d2h, ho.numel()), ("h2d+d2h", both, tot + ho.numel()),
                         ("h2d+d2h pieces", both_pieces, tot + sum(opieces)),
                         ("h2d+d2h per layer", both_layer, tot + sum(opieces)),
                         ("h2d+d2h interleaved (e2e pattern)", both_interleaved, tot + sum(opieces))):
        t = timed(fn)
        print(f"{name}: {t * 1e3:.2f} ms, {nb / t / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
