"""BASELINE.json's five workloads as plain data (SURVEY.md §8a conventions).

Pure Python with no imports from the product package, so that ``bench.py --impl reference``
can read its configuration without loading ``libssbh_cuda.so``. The product package
re-exports this table as ``paper_2308_02856_b200.CONFIGS``.

Seeds: integer N -> MasterSeed::from_hex("%064x" % N); input 1
(config 2: 11), sampling 2, hash 3. ``per_block``: KeyedStream(hash, "hash-seed", j) per
block (config 4), else one shared seed stream (sub 0).
"""

CONFIGS = {
    1: dict(n=1 << 20, s=64, k=8192, p=0.5, seed_in=1, seed_samp=2, seed_hash=3, per_block=False),
    2: dict(n=1 << 24, s=256, k=32768, p=0.3, seed_in=11, seed_samp=2, seed_hash=3,
            per_block=False),
    3: dict(n=1 << 30, s=1024, k=1 << 19, p=0.5, seed_in=1, seed_samp=2, seed_hash=3,
            per_block=False),
    4: dict(n=1 << 34, s=16384, k=3 << 18, p=0.4, seed_in=1, seed_samp=2, seed_hash=3,
            per_block=True),
    5: dict(n=1 << 37, s=32768, k=1 << 21, p=0.5, seed_in=1, seed_samp=2, seed_hash=3,
            per_block=False),
}
