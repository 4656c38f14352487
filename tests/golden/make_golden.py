"""Generates tests/golden/splitmix64_kat.json.

Independent big-integer evaluation of the reference generator
(/root/reference/proj/include/rpchol/rng.hpp:27-42): state += 0x9e3779b97f4a7c15,
z = state; z = (z ^ z>>30) * 0xbf58476d1ce4e5b9; z = (z ^ z>>27) * 0x94d049bb133111eb;
return z ^ z>>31 (all mod 2^64); next_double = (z >> 11) * 2^-53.
No project code is used, so the fixture pins both the oracle and the CUDA path.
Run:  python tests/golden/make_golden.py
"""
import json
import os

M = (1 << 64) - 1


def draws(seed, n):
    s, out = seed, []
    for _ in range(n):
        s = (s + 0x9E3779B97F4A7C15) & M
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        out.append(z ^ (z >> 31))
    return out


def main():
    kat = {}
    for seed in (0, 1, 42, 4242, 0xFFFFFFFFFFFFFFFF):
        d = draws(seed, 16)
        kat[str(seed)] = {
            "u64_hex": [f"{z:016x}" for z in d],
            "u01": [float.hex((z >> 11) * 2.0 ** -53) for z in d],
        }
    # far-counter draws (round 50 of b=200: counters near 2*50*200)
    far = {str(n): f"{draws(7, n + 1)[-1]:016x}" for n in (999, 20000)}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "splitmix64_kat.json")
    with open(path, "w") as f:
        json.dump({"seeds": kat, "seed7_draw_n": far}, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
