"""Counter-based uniform generator shared (as a specification) by the tests and libsem's
`sem_fill_random_state` (which implements the same splitmix64 finaliser in CUDA).

u(seed, box, field, id) in [-1, 1):
    z = seed * 0xD1B54A32D192ED03 + box * 0x8CB92BA72F3D8DD7 + field * 0x9E3779B97F4A7C15
    z += (id + 1) * 0x9E3779B97F4A7C15
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9 ; z = (z ^ (z >> 27)) * 0x94D049BB133111EB ; z ^= z >> 31
    u = 2 * (z >> 11) * 2^-53 - 1        (all arithmetic mod 2^64; id = lexicographic node id)
No method arithmetic: this only produces seeded random fields for operator tests.
"""
import numpy as np

_M = np.uint64


def cb_uniform(seed, box, field, ids):
    ids = np.asarray(ids, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (_M(seed) * _M(0xD1B54A32D192ED03) + _M(box) * _M(0x8CB92BA72F3D8DD7)
             + _M(field) * _M(0x9E3779B97F4A7C15))
        z = z + (ids + _M(1)) * _M(0x9E3779B97F4A7C15)
        z = (z ^ (z >> _M(30))) * _M(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _M(27))) * _M(0x94D049BB133111EB)
        z = z ^ (z >> _M(31))
    return 2.0 * ((z >> _M(11)).astype(np.float64) * 2.0 ** -53) - 1.0
