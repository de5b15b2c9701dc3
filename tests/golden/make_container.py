"""Write small LIFE containers with the REFERENCE package (io.save) so the
container tests pin byte-level compatibility without /root/reference:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \\
        python tests/golden/make_container.py
"""
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
import lifespmv as L  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
for name, dims, mrl, noise, sort in (("ref_small.life", (12, 30, 20, 8, 400), 4.0, 0.1, False),
                                     ("ref_sorted.life", (7, 15, 9, 16, 120), 2.0, 0.0, True)):
    p = L.generate(L.GenConfig(dims=L.Dims(*dims), mean_run_length=mrl, noise_sigma=noise, seed=5))
    if sort:
        t, _ = L.sort_by(p.tensor, "voxel")
        p = L.datagen.Problem(tensor=t, dictionary=p.dictionary, y=p.y, w_true=None, config=None)
    L.io.save(p, os.path.join(OUT, name))
    print("wrote", name, os.path.getsize(os.path.join(OUT, name)))
