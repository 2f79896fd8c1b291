"""Full-launch parity table (the launches tests/test_config_parity_gpu.py
pins): every view of a BASELINE configuration in one device launch, an evenly
spaced sample of views compared with the reference (oracle/_ref) Double —
rel-L2 / max|d|/max|ref| for exact and relaxed, P and BP. Markdown to stdout.
Test infrastructure (reads oracle/_ref as the checker)."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))

from oracle.pyoracle import Reference  # noqa: E402
import test_config_parity_gpu as T  # noqa: E402

CASES = [
    ("c3 512^3, 496 v (bench launch)", T.C3, list(range(0, 496, 62)), ("exact", "relaxed")),
    ("c2 256^3, 248 v / 200 deg",
     ((256, 256, 256), (0.18, 0.18, 0.18), 480, 616, 0.154, 0.154, 749.0, 1198.0, 248, 200.0),
     [0, 62, 124, 186, 247], ("exact", "relaxed")),
    ("c4 512^3 @0.5, 1024^2, SID 300, 360 v",
     ((512, 512, 512), (0.5, 0.5, 0.5), 1024, 1024, 1.0, 1.0, 300.0, 500.0, 360, 360.0),
     [0, 45, 180, 315], ("exact", "relaxed")),
]

if __name__ == "__main__":
    ref = Reference()
    print("| config | sampled views | precision | P rel-L2 / max | BP rel-L2 / max |")
    print("|---|---|---|---|---|")
    for name, cfg, idx, precs in CASES:
        out = T._full_launch_parity(ref, cfg, idx, precisions=precs)
        for p in precs:
            (pa, pb), (ba, bb) = out[p, "P"], out[p, "BP"]
            print(f"| {name} | {len(idx)} | {p} | {pa:.2e} / {pb:.2e} | {ba:.2e} / {bb:.2e} |", flush=True)
