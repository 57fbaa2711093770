"""Epoch permutation pi_{k,e} (reading R10).

The paper never states how clients shuffle (P:209 only says clients "finish
training"); we fix a counter-based generator that both sides implement
independently: SplitMix64's finaliser (Steele, Lea & Flood 2014).

  mix64(z): z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27;
            z *= 0x94D049BB133111EB; z ^= z>>31            (mod 2^64)
  s_{k,e} = mix64(mix64(mix64(seed ^ round) ^ id_k) ^ e)
  key_i   = mix64(s_{k,e} + i * 0x9E3779B97F4A7C15 mod 2^64)
  pi      = indices i in [0, n) stably sorted by key_i ascending.
"""
M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def mix64(z: int) -> int:
    z &= M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M64
    z ^= z >> 31
    return z


def splitmix64_stream(state: int, count: int):
    """The reference SplitMix64 generator: state += golden; out = mix64(state)."""
    out = []
    for _ in range(count):
        state = (state + GOLDEN) & M64
        out.append(mix64(state))
    return out


def epoch_seed(seed: int, rnd: int, client_id: int, epoch: int) -> int:
    return mix64(mix64(mix64((seed ^ rnd) & M64) ^ client_id) ^ epoch)


def epoch_perm(n: int, seed: int, rnd: int, client_id: int, epoch: int) -> list:
    s = epoch_seed(seed, rnd, client_id, epoch)
    keys = [mix64(s + i * GOLDEN) for i in range(n)]
    return sorted(range(n), key=lambda i: keys[i])  # Python's sort is stable
