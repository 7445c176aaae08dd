"""(Needs a -DFHEGPU_ABLATE=1 build of libfhegpu.so, FHEGPU_LIB=...: release kernels compile the ablation bits out.)
Timing ablation of the level kernel: skip stages via debug bits (results invalid)."""
import sys
import numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1611_08769_b200 import DEFAULT_PARAMS, GswScheme, GpuEngine, and_, xor_
lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
s = GswScheme(DEFAULT_PARAMS); keys = s.keygen(1)
rng = np.random.default_rng(1)
eng = GpuEngine(s, keys=keys, rng=rng, batch_size=lanes, device_encrypt=True)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); s.ctx.use_torch_stream(stream)
a, b = eng.input_block(rng.integers(0, 2, (lanes, 2)))
x = xor_(a, b); y = and_(a, b)
prog = eng.flush(); torch.cuda.synchronize()
variants = [(0, "full"), (4, "v2 kernel"), (16, "no A build"), (32, "no B build"), (48, "no A, no B"),
            (64, "no epi math"), (128, "no MMA"), (256, "no loads"), (512, "no stores"),
            (768, "no loads/stores"), (16 | 32 | 64 | 128, "no compute (A,B,MMA,epi)"),
            (16 | 32 | 64 | 128 | 256 | 512, "skeleton only"),
            (4096, "no tile LDTM"), (4096 | 1008, "skeleton, no tile LDTM"),
            (4096 | 16, "no LDTM, no A")]
for dbg, name in variants:
    s.ctx.set_debug(dbg)
    for _ in range(2): prog.run(lanes)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5): prog.run(lanes)
    e1.record(stream); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name:28s} dbg={dbg:4d} ms/step={ms:7.3f}  NAND/s={6*lanes/ms/1e3:7.1f}M  us/item/SM={ms*1e3*148/(6*lanes):.3f}", flush=True)
s.ctx.set_debug(0)
