"""Build a variant of the library with extra -D flags (dev experiments, not product):
    python tools/variant_lib.py OUT.so -DMISA_REF_GROUPS=8
and time one MISA-dagger layer with it on the GPU:
    python tools/variant_lib.py --run OUT.so"""
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

if sys.argv[1] == "--run":
    from paper_2605_07363_b200 import _lib
    _lib.load(sys.argv[2])
    import torch
    from paper_2605_07363_b200 import IndexerEngine, prepare_inputs
    L = 131072
    g = torch.Generator(device="cuda").manual_seed(0)
    K = torch.randn(L, 128, device="cuda", generator=g).bfloat16()
    Q = torch.randn(L, 64, 128, device="cuda", generator=g).bfloat16()
    W = torch.softmax(torch.randn(L, 64, device="cuda", generator=g), -1).float()
    x = prepare_inputs(K, Q, W)
    for method in ("misa", "dsa", "misa_hier"):
        eng = IndexerEngine(method)
        for _ in range(2):
            eng.run_prepared(x)
        st = {}
        for _ in range(3):
            eng.stage_events = []
            eng.run_prepared(x)
            torch.cuda.synchronize()
            ev = eng.stage_events
            for (n0, e0), (_, e1) in zip(ev, ev[1:]):
                st[n0] = st.get(n0, 0.0) + e0.elapsed_time(e1) / 3
        print(sys.argv[2], method, {k: round(v, 3) for k, v in st.items()}, flush=True)
        del eng
else:
    from paper_2605_07363_b200 import _build
    out, flags = sys.argv[1], sys.argv[2:]
    objs = []
    for src in _build.SOURCES:
        o = f"/tmp/variant_{src}.o"
        subprocess.check_call([_build._nvcc(), *_build.ARCH, *_build.FLAGS, *flags, "-c",
                               os.path.join(_build.CSRC, src), "-o", o])
        objs.append(o)
    subprocess.check_call([_build._nvcc(), *_build.ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", out, *objs,
                           "-cudart", "static"])
    print(out)
