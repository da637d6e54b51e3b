"""Static SMEM bank-conflict check of the JIT pass kernels (dev tool, CPU only):
reads each mapping's lane offsets from the emitted PTX prologue and counts the
wavefronts of a warp's 64-bit access (16-lane phases) with the flip vector 0."""
import re
import sys

sys.path.insert(0, ".")
from paper_2504_03967_b200 import statevec as sv  # noqa: E402
from paper_2504_03967_b200.generators import RandomSpec, qft_arrays, random_arrays  # noqa: E402


def wavefronts(offs):
    wf = 0
    for half in (0, 1):
        banks = {}
        for l in range(16):
            lane = l + 16 * half
            a = 0
            for b in range(5):
                if lane >> b & 1:
                    a ^= offs[b]
            banks.setdefault((a >> 3) & 15, set()).add(a)
        wf += max(len(v) for v in banks.values())
    return wf


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    kind = sys.argv[2] if len(sys.argv) > 2 else "random"
    gt, gp = random_arrays(RandomSpec(n, 1000, 0)) if kind == "random" else qft_arrays(n)
    p = sv.CompiledCircuit(gt, gp, n, "fp32", jit=-1)
    tot = bad = 0
    for i in range(p.info["n_passes"]):
        lines = p.pass_ptx(i).split("\n")
        vals = []
        for j, ln in enumerate(lines):
            m = re.match(r"\s*and.b32 %r\d+, %r\d+, (\d+);", ln)
            if m and "neg.s32" in lines[j - 1]:
                vals.append(int(m.group(1)))
            if "bar.sync" in ln:
                break
        wb = 3
        maps = [vals[k:k + 5] for k in range(0, len(vals), 5 + wb)]
        w = [wavefronts(m) for m in maps]
        tot += len(w)
        bad += sum(1 for x in w if x > 2)
    print(f"{kind} n={n}: passes {p.info['n_passes']} mappings {tot} conflicted {bad}")


if __name__ == "__main__":
    main()
