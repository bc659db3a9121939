"""Phase timing of the v3 encoder (thread-0 clock64 deltas per block).

Builds a variant library with -DAPAX_V3_PROF under build_variants/ (the
product .so is untouched), runs the cfg2 workload and prints the mean
cycles per block of each phase: S1 / phase B / FQ update+phase C / resolve
+phase D / phase A(next) / flush+bookkeeping / unit end."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1303_4994_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "build_variants")
SO = os.path.join(OUT, "libapax_prof.so")


def build(defs=("-DAPAX_V3_PROF",), so=None):
    so = so or SO
    os.makedirs(OUT, exist_ok=True)
    src = os.path.join(ROOT, "paper_1303_4994_b200", "csrc")
    objs = []
    for f in ["apax_encode.cu", "apax_encode_v2.cu", "apax_encode_v3.cu", "apax_decode.cu", "apax_decode_v2.cu",
              "apax_decode_v3.cu", "apax_profile.cu", "apax_k5.cu", "apax_capi.cu"]:
        o = os.path.join(OUT, f.replace(".cu", ".o"))
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
                        "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", *defs,
                        "-c", os.path.join(src, f), "-o", o], check=True)
        objs.append(o)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", so]
                   + objs, check=True)


def main():
    if "--build" in sys.argv:
        build()
        return
    if "--variant" in sys.argv:   # --variant NAME -DX -DY ...: build_variants/libapax_NAME.so
        i = sys.argv.index("--variant")
        name, defs = sys.argv[i + 1], sys.argv[i + 2:]
        build(tuple(defs), os.path.join(OUT, f"libapax_{name}.so"))
        return
    seg = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    L = ctypes.CDLL(SO)
    n = 1 << 26
    x = torch.from_numpy(W.cfg2_ar2_f32(n)).cuda()
    bs = 4096
    nb = n // bs
    L.apax_max_encoded_bytes.restype = ctypes.c_int64
    L.apax_encode_workspace_bytes.restype = ctypes.c_int64
    cap = L.apax_max_encoded_bytes(ctypes.c_int64(n), 3, bs)
    wsb = L.apax_encode_workspace_bytes(ctypes.c_int64(n), 3, 2, bs, ctypes.c_int64(seg))
    out = torch.empty(cap + 64, dtype=torch.uint8, device="cuda")
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    st = torch.empty(4, dtype=torch.int64, device="cuda")
    offs = torch.empty(nb + 1, dtype=torch.int64, device="cuda")
    tr = torch.zeros(nb * 10 + 8, dtype=torch.float64, device="cuda")
    for it in range(3):
        tr.zero_()
        r = L.apax_encode(ctypes.c_void_p(x.data_ptr()), ctypes.c_int64(n), 3, 2, ctypes.c_double(W.CFG2_TARGET_DB),
                          bs, ctypes.c_int64(seg), 0, ctypes.c_void_p(out.data_ptr()), ctypes.c_int64(cap),
                          ctypes.c_void_p(offs.data_ptr()), ctypes.c_void_p(st.data_ptr()),
                          ctypes.c_void_p(tr.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ctypes.c_int64(wsb), None)
        assert r == 0, r
        torch.cuda.synchronize()
    acc = tr[nb * 10:].view(torch.int64).cpu().tolist()
    names = ["S1", "phaseB", "FQupd+phaseC", "resolve+D", "phaseA(next)", "flush+book", "unit end/start", "[stage wait]"]
    tot = sum(acc[:7])
    print(f"segment_blocks={seg}: cycles per block per CTA (sum over CTAs / blocks)")
    for nm, v in zip(names, acc):
        print(f"  {nm:16s} {v / nb:10.0f}  ({v / tot * 100:5.1f}%)")
    print(f"  total            {tot / nb:10.0f}")


if __name__ == "__main__":
    main()
