"""Write tests/golden/synth_golden.txt from a pure-Python-int rendering of the
generator spec in synth/gen.py's docstring.  Calls neither the
CUDA path nor numpy; the test checks synth.gen_block (numpy) and the CUDA twin
against these bits."""
import os
import struct

M64 = (1 << 64) - 1


def splitmix64(x):
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def bf16_rne(f):
    u = struct.unpack("<I", struct.pack("<f", f))[0]
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF


def value(seed, tensor, dist, layer, head, pos, dim):
    if dist == "ONE" and tensor == 2:
        return 0x3F80
    if dist == "S" and tensor == 1 and pos == 0:
        return 0x3F80
    key = ((((tensor * 128 + layer) * 128 + head) << 23 | pos) << 8) | dim
    h = splitmix64(key ^ ((seed * 0x9E3779B97F4A7C15) & M64))
    v = (h >> 40) - (1 << 23)
    scale = 16.0 if (dist == "P" and tensor == 0) else 1.0
    x = v * 2.0 ** -23 * scale          # exact in binary64 and in fp32
    if dist == "S" and tensor == 0:
        x = abs(x)
    return bf16_rne(x)


CASES = [
    (0x48454144, t, dist, layer, head, pos, dim)
    for dist in ("U", "P", "S", "ONE")
    for (t, layer, head, pos, dim) in [
        (0, 0, 0, 0, 0), (0, 0, 3, 17, 63), (1, 0, 1, 0, 5), (1, 31, 7, 1048575, 127),
        (2, 79, 7, 4194303, 100), (2, 2, 0, 1, 0), (0, 31, 31, 1048576, 127), (1, 5, 2, 0, 0),
    ]
] + [(s, 0, "U", 0, 0, 3, 7) for s in (0, 1, 7, 123456789)]

if __name__ == "__main__":
    path = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "synth_golden.txt")
    with open(path, "w") as f:
        f.write("# seed tensor dist layer head pos dim bf16_bits(hex)\n")
        f.write("# written by tools/make_synth_golden.py (pure-Python-int rendering of the SURVEY.md §8(d) spec)\n")
        for c in CASES:
            f.write(" ".join(str(x) for x in c) + f" {value(*c):04x}\n")
    print("wrote", len(CASES), "cases")
