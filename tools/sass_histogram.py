"""SASS opcode histograms of the headline executor instantiations (static
instruction counts from cuobjdump of the built library): the evidence of which
data-movement instructions each kernel uses (LDGSTS = cp.async, UTMALDG /
UBLKCP = TMA, LDS/STS shared, LDG/STG global, BAR, RED/ATOM).

    python tools/sass_histogram.py > profiles/r02/sass_histogram.md
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_1802_03749_b200" / "lib" / "libmeshplan_b200.so"
# (label, demangled-name fragments that must all appear)
KERNELS = [
    ("C5 / C1 headline: hier_stream_kernel<OpFlux, double, AoS, colour, u8 slots, push>",
     ["hier_stream_kernel", "OpFluxEdLi0ELb0EhLi2ELb0ELb1ELb0ELb0EEEv"]),
    ("C5 pull form: hier_stream_kernel<OpFlux, double, ..., PULL>", ["hier_stream_kernel", "OpFluxEdLi0ELb0EhLi2ELb0ELb1ELb1ELb0EEEv"]),
    ("multi-GPU fused export: hier_stream_kernel<OpFlux, double, ..., push, EXPORT>",
     ["hier_stream_kernel", "OpFluxEdLi0ELb0EhLi2ELb0ELb1ELb0ELb1EEEv"]),
    ("C2 headline: hier_stream_kernel<OpFlux, float, AoS, colour, u8 slots, push>",
     ["hier_stream_kernel", "OpFluxEfLi0ELb0EhLi2ELb0ELb1ELb0ELb0EEEv"]),
    ("C3 headline: hier_stream_kernel<OpScatter8, double, AoS, colour, u16 slots, 4 rows/thread>",
     ["hier_stream_kernel", "OpScatter8EdLi0ELb0EtLi4E"]),
    ("gather form: hier_gather_kernel<OpFlux, double>", ["hier_gather_kernel", "OpFluxEdh"]),
    ("C4 headline: hier_pipe_kernel<OpFaceFlux, double, AoS, colour, pull>",
     ["hier_pipe_kernel", "OpFaceFluxEdLi0ELb0E", "Lb1EEEv"]),
    ("global colouring baseline: global_colour_kernel<OpFlux, double>", ["global_colour_kernel", "OpFlux", "Ed"]),
    ("atomics baseline: atomic_kernel<OpFlux, double>", ["atomic_kernel", "OpFlux", "Ed"]),
    ("block colouring: greedy_blocks_kernel<2>", ["greedy_blocks_kernel", "ILi2E"]),
    ("halo put (peer memory): halo_put_kernel<double>", ["halo_put_kernel", "IdE"]),
    ("halo get (peer memory): halo_get_kernel<double>", ["halo_get_kernel", "IdE"]),
]
CLASSES = {"LDGSTS": "cp.async gather", "UTMALDG": "TMA tensor load", "UBLKCP": "TMA bulk copy", "LDS": "shared load",
           "STS": "shared store", "LDG": "global load", "STG": "global store", "BAR": "barrier", "RED": "reduction",
           "ATOM": "atomic", "ATOMS": "shared atomic", "SYNCS": "mbarrier", "DMUL": "fp64 mul", "DADD": "fp64 add",
           "SHFL": "shuffle", "REDUX": "warp reduce", "MEMBAR": "fence", "LDGDEPBAR": "cp.async commit",
           "DEPBAR": "cp.async wait", "ACQBULK": "bulk/PDL", "CCTL": "cache control"}


def functions(sass: str):
    cur, body = None, []
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur:
            body.append(line)
    if cur:
        yield cur, body


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    funcs = list(functions(sass))
    print("# SASS opcode histograms (static counts, sm_100a, `cuobjdump -sass` of libmeshplan_b200.so)\n")
    for label, frags in KERNELS:
        hits = [(n, b) for n, b in funcs if all(f in n for f in frags)]
        if not hits:
            print(f"## {label}\n\n(not found)\n")
            continue
        name, body = min(hits, key=lambda nb: len(nb[0]))
        ops = collections.Counter()
        wide = collections.Counter()  # 256-bit global accesses (LDG/STG.E.ENL2.256)
        for line in body:
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
            if m:
                ops[m.group(1)] += 1
                if m.group(2) and "ENL2.256" in m.group(2):
                    wide[m.group(1)] += 1
        total = sum(ops.values())
        print(f"## {label}\n\n`{name[:160]}`\n\n{total} instructions.  Data movement / sync:\n")
        print("| opcode | what | count |\n|---|---|---|")
        for op in sorted(ops, key=lambda o: -ops[o]):
            if op in CLASSES:
                extra = f" ({wide[op]} of them 256-bit `.ENL2.256`)" if wide[op] else ""
                print(f"| {op} | {CLASSES[op]} | {ops[op]}{extra} |")
        others = ", ".join(f"{o} {c}" for o, c in ops.most_common(12) if o not in CLASSES)
        print(f"\nMost frequent others: {others}\n")


if __name__ == "__main__":
    sys.exit(main())
