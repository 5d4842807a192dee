import sys
sys.path.insert(0, ".")
from tools.prefill_bench import run  # noqa: E402
for T in (16, 32, 64, 128, 256):
    print("T", T, end=": ")
    run(1, 8192, 8192, T=T)
for g in ((32, 32), (32, 4), (32, 8)):
    print("Hq,Hkv", g, end=": ")
    run(1, 8192, 8192, Hq=g[0], Hkv=g[1], T=128)
