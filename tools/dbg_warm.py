import sys, numpy as np, torch, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import GOLDEN, load_container
from paper_1303_4994_b200 import encode_device, StreamConfig, Dtype, Mode
name = sys.argv[1] if len(sys.argv) > 1 else "warm_cfg1_fr4_P4"
c = load_container(GOLDEN / "containers" / (name + ".npz"))
m = c["meta"]
DT = {"i8": Dtype.I8, "i16": Dtype.I16, "i32": Dtype.I32, "f32": Dtype.F32, "f64": Dtype.F64}
POL = {0: "cold", 1: "warm_self"}
cfg = StreamConfig(DT[m["dtype"]], m["block_size"], Mode(m["mode"]), float.fromhex(m["target_hex"]),
                   segment_blocks=m["segment_blocks"] or None, segment_policy=POL[m["policy"]])
print(m)
x = torch.from_numpy(np.ascontiguousarray(c["x"])).cuda()
r = encode_device(x, cfg)
got, ref = r.to_bytes(), c["blob"]
print(len(got), len(ref), got == ref)
offs = r.block_offsets.cpu().numpy(); print("offs", offs.tolist()); print("ref ", c["offsets"].tolist())
n = min(len(got), len(ref))
d = next((i for i in range(n) if got[i] != ref[i]), None)
print("first diff", d)
