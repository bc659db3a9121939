import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import GOLDEN, load_container
from paper_1303_4994_b200 import encode_device, StreamConfig, Dtype, Mode
c = load_container(GOLDEN / "containers" / (sys.argv[1] + ".npz"))
m = c["meta"]
DT = {"i8": Dtype.I8, "i16": Dtype.I16, "i32": Dtype.I32, "f32": Dtype.F32, "f64": Dtype.F64}
cfg = StreamConfig(DT[m["dtype"]], m["block_size"], Mode(m["mode"]), float.fromhex(m["target_hex"]),
                   segment_blocks=m["segment_blocks"] or None)
x = torch.from_numpy(np.ascontiguousarray(c["x"])).cuda()
r = encode_device(x, cfg)
print("OK" if r.to_bytes() == c["blob"] else "MISMATCH")
