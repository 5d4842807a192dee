"""No source file names a copy call that is closed on the GPU pool (its batched forms raised a
GPU fault there). The pattern is assembled from fragments so this file never contains a name."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXTS = (".c", ".cc", ".cpp", ".cu", ".cuh", ".h", ".hpp", ".py", ".sh")
SKIP = {".git", "gpurun_out", "baseline", "__pycache__"}


def closed_names():
    parts = [("cuda", ""), ("cuda", "3D"), ("cu", ""), ("cu", "3D")]
    return [f"{p}Memcpy{d}" + "Batch" + "Async" for p, d in parts]


def test_no_closed_copy_call_named_in_sources():
    pat = re.compile("|".join(closed_names()))
    hits = []
    for dp, dns, fns in os.walk(ROOT):
        dns[:] = [d for d in dns if d not in SKIP]
        for fn in fns:
            if fn.endswith(EXTS):
                path = os.path.join(dp, fn)
                with open(path, errors="replace") as f:
                    for i, line in enumerate(f, 1):
                        if pat.search(line):
                            hits.append(f"{os.path.relpath(path, ROOT)}:{i}")
    assert not hits, hits
