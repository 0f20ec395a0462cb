"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every kernel
and every integrand MODE on tiny links (multi-class spans, mixed rates with gaps in the lattice
lines, two line segments per region, coherent regions, shards + combine).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2412_11614_b200 as isrs
    from workloads import tiny_link
    links = [
        tiny_link(n_ch=3, rates_gbd=(64, 32), guard_ghz=20.0, n_span=4, grid_n=8, random_spans=True,
                  fmts=("16qam", "gauss")),
        tiny_link(n_ch=5, rates_gbd=(32, 64, 96), guard_ghz=12.5, n_span=2, grid_n=8,
                  fmts=("qpsk", "16qam", "64qam")),
        tiny_link(n_ch=2, rates_gbd=(65,), spacing_ghz=100.0, n_span=1, grid_n=260, fmts=("qpsk",)),
        tiny_link(n_ch=3, rates_gbd=(96,), spacing_ghz=100.0, n_span=12, grid_n=8, fmts=("16qam",)),
    ]
    opts = [dict(), dict(precision=32), dict(flags=isrs.FLAG_DEDUP), dict(flags=isrs.FLAG_LITERAL_GAIN),
            dict(mu_mode=isrs.MU_MACLAURIN), dict(f_samples=2), dict(flags=isrs.FLAG_NO_CHAIN),
            dict(flags=isrs.FLAG_SPLIT), dict(flags=isrs.FLAG_MIRROR)]
    n = 0
    for li, link in enumerate(links):
        for o in (opts if li != 2 else opts[:1]):
            with isrs.Engine(link, **o) as e:
                eta, _ = e.nli(terms=True)
                if o.get("flags") == isrs.FLAG_SPLIT:
                    e.nli_split()
                torch.cuda.synchronize()
                assert torch.isfinite(eta).all()
                n += 1
    # integral form (one small link) and the shard path
    with isrs.Engine(links[1], mu_mode=isrs.MU_INTEGRAL) as e:
        e.nli(coi=[2])
        torch.cuda.synchronize()
    with isrs.Engine(links[0]) as e:
        parts = torch.stack([e.nli_shard(r, 2) for r in range(2)])
        e.combine(parts)
        torch.cuda.synchronize()
    print(f"sanitize_run ok: {n + 2} handles", flush=True)


if __name__ == "__main__":
    main()
