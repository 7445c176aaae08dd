"""Config-level GPU parity: ciphertexts gate by gate and decrypted outputs vs the reference.

Golden digests come from running the reference itself (tests/golden/make_golden.py);
the gate-by-gate chain covers every hom_nand / hom_not the reference evaluated, in order.
"""

import os

import numpy as np
import pytest

from oracle import digest
from paper_1611_08769_b200 import (DEFAULT0_PARAMS, DEFAULT_PARAMS, EXACT_PARAMS, FixedFormat,
                                   GpuEngine, GswScheme, and_, fft_1d, fft_2d, input_signal, xor_)
from paper_1611_08769_b200.fft import read_signal_ints, signal_words
from tests.helpers import GOLDEN, FFT_CONFIGS, config_signal, golden_json, golden_npz, model_outputs

pytestmark = pytest.mark.gpu

PARAMS = {"EXACT": EXACT_PARAMS, "DEFAULT0": DEFAULT0_PARAMS}


def gate_digests(eng, lane=0, chunk=16384):
    """Digest of every hom_nand / hom_not output in reference order, plus input digests."""
    trace = eng.trace
    ins = [t for t in trace if t[0] == 2]
    gates = [t for t in trace if t[0] in (0, 1)]

    def digs(entries):
        out = []
        for s in range(0, len(entries), chunk):
            part = entries[s:s + chunk]
            vals = eng.read_nodes([t[4] for t in part], [t[5] for t in part], lanes=[lane])
            out.extend(digest.digest_compact(v[0]) for v in vals)
        return out
    return digs(ins), digs(gates)


def run_fft_config(cfg, device_encrypt, keep_all=True, lanes=1, schedule="levels"):
    pname, seed, (F, f), dims, _ = FFT_CONFIGS[cfg]
    params = PARAMS[pname]
    scheme = GswScheme(params)
    keys = scheme.keygen(seed)
    if lanes == 1:
        rng, x = config_signal(cfg)
        eng = GpuEngine(scheme, keys=keys, rng=rng, keep_all=keep_all, record_trace=keep_all,
                        device_encrypt=device_encrypt, schedule=schedule)
        values = x
    else:
        rngs, vals = [], []
        for lane in range(lanes):
            r, x = config_signal(cfg, lane)
            rngs.append(r)
            vals.append(x)
        eng = GpuEngine(scheme, keys=keys, batch_size=lanes, lane_rngs=rngs,
                        device_encrypt=device_encrypt, keep_all=keep_all, record_trace=keep_all,
                        schedule=schedule)
        values = np.array(vals)
    sig = input_signal(eng, values, FixedFormat(F, f), dims=dims if isinstance(dims, tuple) else None)
    out = fft_2d(sig) if isinstance(dims, tuple) else fft_1d(sig)
    eng.flush()
    return eng, out, values


@pytest.mark.parametrize("device_encrypt", [False, True], ids=["host-enc", "device-enc"])
def test_cfg0_gate_by_gate(device_encrypt):
    eng, out, x = run_fft_config("cfg0", device_encrypt)
    ref = golden_json("cts_cfg0.json")
    ins, gates = gate_digests(eng)
    assert digest.chain_digest(ins) == ref["inputs_chain"]
    gd = golden_npz("cts_cfg0.npz")["gate_digests"].view(np.uint8).reshape(-1, 8)
    want = [bytes(r).hex() for r in gd]
    first_bad = next((i for i, (a, b) in enumerate(zip(gates, want)) if a != b), None)
    assert first_bad is None, f"first differing gate {first_bad}"
    assert digest.chain_digest(gates) == ref["gates_chain"]
    assert read_signal_ints(eng, out)[0].tolist() == ref["output_words"]
    assert (eng.nand_count, eng.max_depth) == (ref["nand_count"], ref["max_depth"])


@pytest.mark.parametrize("schedule", ["flow", "auto"])
def test_cfg0_flow_gate_by_gate(schedule):
    """configs[0] as ONE warp-dataflow launch (csrc/flow_nand.cuh; 'auto' picks it for deep
    single-lane EXACT programs): every gate's ciphertext equals the reference's, and stays so
    over repeated runs of the same program (the scratch tags advance with every run)."""
    eng, out, x = run_fft_config("cfg0", True, schedule=schedule)
    assert eng.last_compile["schedule"] == "flow" and eng.last_program.launches == 1
    assert min(eng.last_compile["flow"][k] for k in ("ring_operands", "scratch_operands", "store_operands")) > 0
    ref = golden_json("cts_cfg0.json")
    gd = golden_npz("cts_cfg0.npz")["gate_digests"].view(np.uint8).reshape(-1, 8)
    want = [bytes(r).hex() for r in gd]
    for runs in (0, 3):
        for _ in range(runs):
            eng.last_program.run(1)
        ins, gates = gate_digests(eng)
        assert digest.chain_digest(ins) == ref["inputs_chain"]
        first_bad = next((i for i, (a, b) in enumerate(zip(gates, want)) if a != b), None)
        assert first_bad is None, f"first differing gate {first_bad} after {runs} reruns"
    assert read_signal_ints(eng, out)[0].tolist() == ref["output_words"]
    assert (eng.nand_count, eng.max_depth) == (ref["nand_count"], ref["max_depth"])


def test_cfg0_flow_epoch_wraps():
    """More runs of one warp-dataflow program than there are scratch tags (32,767): a stale
    row of an earlier run is never taken for the current one."""
    eng, out, x = run_fft_config("cfg0", True, keep_all=False, schedule="flow")
    ref = golden_json("cts_cfg0.json")
    handles = [h for w in signal_words(out) for h in w.bits]
    v0 = eng.node_values(handles)
    for _ in range(32767 + 5):
        eng.last_program.run(1)
    assert np.array_equal(eng.node_values(handles), v0)
    assert read_signal_ints(eng, out)[0].tolist() == ref["output_words"]


def test_cfg1_sample_pairs_bit_exact():
    """First 4096 pairs of the 2^20-pair gate benchmark: every XOR/AND ciphertext."""
    ref = golden_json("cts_cfg1.json")
    pairs = ref["pairs"]
    scheme = GswScheme(DEFAULT_PARAMS)
    keys = scheme.keygen(1)
    rng = np.random.default_rng(1)
    bits = rng.integers(0, 2, (1 << 20, 2))
    eng = GpuEngine(scheme, keys=keys, rng=rng, batch_size=pairs, device_encrypt=True,
                    keep_all=True, record_trace=True)
    a, b = eng.input_block(bits[:pairs])
    x = xor_(a, b)
    y = and_(a, b)
    assert eng.read_back_bits([x])[0].tolist() == (bits[:pairs, 0] ^ bits[:pairs, 1]).tolist()
    assert eng.read_back_bits([y])[0].tolist() == (bits[:pairs, 0] & bits[:pairs, 1]).tolist()
    vx = eng.node_values([x])[0]
    vy = eng.node_values([y])[0]
    assert [digest.digest_compact(v) for v in vx] == ref["xor_digests"]
    assert [digest.digest_compact(v) for v in vy] == ref["and_digests"]
    gates = [t for t in eng.trace if t[0] in (0, 1)]
    assert len(gates) == 6
    vals = eng.read_nodes([t[4] for t in gates], [t[5] for t in gates])     # (6, pairs, N, k)
    per_pair = [digest.digest_compact(vals[g, p]) for p in range(pairs) for g in range(6)]
    assert per_pair[:len(ref["first_gates"])] == ref["first_gates"]
    assert digest.chain_digest(per_pair) == ref["gates_chain"]
    assert eng.nand_count == 6 and eng.max_depth == 3


@pytest.mark.parametrize("schedule", ["auto", "tiled"])
def test_cfg1_sample_outputs_default_schedules(schedule):
    """The same 4096 pairs on the schedules the benchmark uses ('auto' = lane-resident for the
    XOR + AND program, and tiled): every output ciphertext equals the reference's."""
    ref = golden_json("cts_cfg1.json")
    pairs = ref["pairs"]
    scheme = GswScheme(DEFAULT_PARAMS)
    keys = scheme.keygen(1)
    rng = np.random.default_rng(1)
    bits = rng.integers(0, 2, (1 << 20, 2))
    eng = GpuEngine(scheme, keys=keys, rng=rng, batch_size=pairs, device_encrypt=True, schedule=schedule)
    a, b = eng.input_block(bits[:pairs])
    x, y = xor_(a, b), and_(a, b)
    eng.flush()
    assert eng.last_compile["schedule"] == ("resident" if schedule == "auto" else "tiled")
    vx, vy = eng.node_values([x, y])
    assert [digest.digest_compact(v) for v in vx] == ref["xor_digests"]
    assert [digest.digest_compact(v) for v in vy] == ref["and_digests"]


def test_cfg4_all_lanes_outputs():
    """1024 signals as lanes (device encryption, per-lane generators): all outputs bit-exact."""
    eng, out, vals = run_fft_config("cfg4", device_encrypt=True, keep_all=False, lanes=1024)
    got = read_signal_ints(eng, out)
    want = golden_npz("clear_cfg4.npz")["words"]
    assert np.array_equal(got, want)
    assert np.array_equal(got, model_outputs("cfg4", vals))
    assert eng.nand_count == golden_json("trace_cfg4.json")["nand_count"]
    assert eng.launches == golden_json("trace_cfg4.json")["max_depth"]   # one launch per level


@pytest.mark.parametrize("normalize", [False, True])
def test_ifft_cfg4_geometry_all_lanes(normalize):
    """ifft_1d on the GPU (cfg4 geometry: 1024 lanes of 16-point Q4.12 signals, DEFAULT0,
    device encryption with per-lane generators): every lane's decrypted output equals the
    integer model of swap(fft(swap(x))) (>> log2 M when normalising).  The reference has no
    inverse, so the integer model (oracle/fixedfft.py) is the oracle."""
    from oracle import fixedfft
    from paper_1611_08769_b200.fft import ifft_1d
    scheme = GswScheme(DEFAULT0_PARAMS)
    keys = scheme.keygen(4)
    lanes, M, F, f = 1024, 16, 16, 12
    rngs, vals = [], []
    for lane in range(lanes):
        r, x = config_signal("cfg4", lane)
        rngs.append(r)
        vals.append(x)
    vals = np.array(vals)
    eng = GpuEngine(scheme, keys=keys, batch_size=lanes, lane_rngs=rngs, device_encrypt=True)
    out = ifft_1d(input_signal(eng, vals, FixedFormat(F, f)), normalize=normalize)
    got = read_signal_ints(eng, out)
    re = fixedfft.encode_lanes(vals.real, F, f)
    im = fixedfft.encode_lanes(vals.imag, F, f)
    o_im, o_re = fixedfft.fft_1d(im, re, F, f)
    if normalize:
        o_re, o_im = o_re >> 4, o_im >> 4
    assert np.array_equal(got, fixedfft.interleave(o_re, o_im))
    assert eng.nand_count == golden_json("trace_cfg4.json")["nand_count"]


def test_cfg4_lane0_gate_by_gate():
    eng, out, _ = run_fft_config("cfg4", device_encrypt=True)
    ref = golden_json("cts_cfg4.json")
    ins, gates = gate_digests(eng)
    assert digest.chain_digest(ins) == ref["inputs_chain"]
    every = ref["checkpoint_every"]
    cps = [digest.chain_digest(gates[:i]) for i in range(every, len(gates) + 1, every)]
    assert cps == ref["gates_checkpoints"]
    assert digest.chain_digest(gates) == ref["gates_chain"]
    assert read_signal_ints(eng, out)[0].tolist() == ref["output_words"]


@pytest.mark.parametrize("cfg,schedule", [("cfg3", "levels"), ("cfg3", "dataflow"), ("cfg3", "queue"),
                                          ("cfg2", "levels"), ("cfg2", "dataflow"), ("cfg2", "queue")])
def test_fft_config_gate_by_gate(cfg, schedule):
    """Every gate's ciphertext equals the reference's; 'dataflow' runs the whole FFT as one
    launch with per-operand readiness (SSA slots, per-CTA progress counters), 'queue' as one
    launch over a ready queue (CTAs pop items whose producers have completed)."""
    path = os.path.join(GOLDEN, f"cts_{cfg}.json")
    if not os.path.exists(path):
        pytest.skip(f"golden {cfg} ciphertext digests not generated")
    eng, out, x = run_fft_config(cfg, device_encrypt=True, schedule=schedule)
    if schedule == "dataflow":
        assert eng.launches == 1                      # one launch for the whole FFT
    elif schedule == "queue":
        assert eng.launches == 2                      # queue reset + one launch for the whole FFT
    ref = golden_json(f"cts_{cfg}.json")
    ins, gates = gate_digests(eng)
    assert digest.chain_digest(ins) == ref["inputs_chain"]
    assert digest.chain_digest(gates) == ref["gates_chain"]
    assert read_signal_ints(eng, out)[0].tolist() == ref["output_words"]
    assert read_signal_ints(eng, out)[0].tolist() == golden_npz(f"clear_{cfg}.npz")["words"][0].tolist()


def test_device_encryption_equals_host_encryption():
    for params, seed in ((DEFAULT_PARAMS, 1), (EXACT_PARAMS, 3)):
        s = GswScheme(params)
        keys = s.keygen(seed)
        r_host = np.random.default_rng(42)
        r_dev = np.random.default_rng(42)
        bits = r_host.integers(0, 2, (3, 6))          # even count: no buffered half left
        r_dev.integers(0, 2, (3, 6))
        host = s.encrypt_many(keys.public_key, bits.ravel(), r_host)
        eng = GpuEngine(s, keys=keys, rng=r_dev, batch_size=3, device_encrypt=True)
        hs = eng.input_block(bits)
        dev = eng.node_values(hs)                                    # (6, 3, N, k)
        assert np.array_equal(dev.transpose(1, 0, 2, 3).reshape(-1, params.n_ct, params.k), host)
        sh, sd = r_host.bit_generator.state, r_dev.bit_generator.state
        assert sh["state"] == sd["state"] and sh["has_uint32"] == sd["has_uint32"] == 0


def test_dataflow_many_lanes_equals_levels():
    """Dataflow (items = (op, lane), CTA-strided) and ready-queue launches with several lanes
    vs level launches."""
    outs = {}
    for schedule in ("levels", "dataflow", "queue"):
        eng, out, vals = run_fft_config("cfg4", device_encrypt=True, keep_all=False, lanes=5,
                                        schedule=schedule)
        outs[schedule] = read_signal_ints(eng, out)
        assert np.array_equal(outs[schedule], model_outputs("cfg4", vals))
    assert np.array_equal(outs["levels"], outs["dataflow"])
    assert np.array_equal(outs["levels"], outs["queue"])


def test_tiled_schedule_equals_levels_bit_exact():
    """schedule='tiled' (auto for wide programs): 4096 XOR+AND pairs in 32 chunks of 128 lanes,
    one wavefront dataflow launch -- every output ciphertext equals the level schedule's."""
    scheme = GswScheme(DEFAULT_PARAMS)
    keys = scheme.keygen(1)
    bits = np.random.default_rng(9).integers(0, 2, (4096, 2))
    outs = {}
    for schedule in ("levels", "tiled"):
        eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(1), batch_size=4096,
                        device_encrypt=True, schedule=schedule)
        a, b = eng.input_block(bits)
        x, y = xor_(a, b), and_(a, b)
        prog = eng.flush()
        assert (prog.tile_lanes == 128) == (schedule == "tiled")
        outs[schedule] = eng.node_values([x, y])
        assert (eng.read_back_bits([x, y]) == np.stack([bits[:, 0] ^ bits[:, 1], bits[:, 0] & bits[:, 1]])).all()
        prog.run(4096)                                     # re-running rewrites identical values
        assert np.array_equal(eng.node_values([x, y]), outs[schedule])
    assert np.array_equal(outs["levels"], outs["tiled"])


@pytest.mark.parametrize("schedule", ["tiled", "resident"])
def test_chained_flushes_equal_levels(schedule):
    """Two chained programs (the second consumes the first's outputs; tiled: its own ring of
    temporaries above every live slot; resident: its own per-lane plan) equal the level
    schedule bit for bit."""
    scheme = GswScheme(DEFAULT0_PARAMS)                # depth 5 > DEFAULT's budget of 3
    keys = scheme.keygen(2)
    bits = np.random.default_rng(4).integers(0, 2, (2048, 3))
    res = {}
    for sched in ("levels", schedule):
        eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(2), batch_size=2048,
                        device_encrypt=True, schedule=sched)
        a, b, c = eng.input_block(bits)
        x, y = xor_(a, b), and_(a, b)
        p1 = eng.flush()
        z, w = xor_(x, c), and_(y, c)                 # second program on the first's outputs
        p2 = eng.flush()
        if sched == "tiled":
            assert p1.tile_lanes == 128 and p2.tile_lanes == 128
        elif sched == "resident":
            assert p1.launches == 1 and p2.launches == 1
        res[sched] = eng.node_values([x, y, z, w])
        got = eng.read_back_bits([z, w])
        assert (got[0] == (bits[:, 0] ^ bits[:, 1] ^ bits[:, 2])).all()
        assert (got[1] == (bits[:, 0] & bits[:, 1] & bits[:, 2])).all()
    assert np.array_equal(res["levels"], res[schedule])


def test_cfg1_full_size_every_lane_decrypts():
    """configs[1] at full size (2^20 pairs, the default lane-resident schedule with a partial
    last 3-lane group, device encryption with the cfg1 seeds): every one of the 2^21 output
    ciphertexts decrypts to the right bit."""
    scheme = GswScheme(DEFAULT_PARAMS)
    keys = scheme.keygen(1)
    rng = np.random.default_rng(1)
    bits = rng.integers(0, 2, (1 << 20, 2))
    eng = GpuEngine(scheme, keys=keys, rng=rng, batch_size=1 << 20, device_encrypt=True)
    a, b = eng.input_block(bits)
    x, y = xor_(a, b), and_(a, b)
    prog = eng.flush()
    assert eng.last_compile["schedule"] == "resident" and prog.launches == 1
    got = eng.read_back_bits([x, y])
    assert (got[0] == (bits[:, 0] ^ bits[:, 1])).all()
    assert (got[1] == (bits[:, 0] & bits[:, 1])).all()
    assert eng.nand_count == 6 and eng.max_depth == 3


def _store_view(ctx, first_ct, count):
    """torch view (count, ct_words) u32 of a store range, on the device (no host copy)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (count, ctx.ct_words), "typestr": "<u4", "version": 3,
                                    "data": (ctx.store_ptr + first_ct * ctx.ct_words * 4, False),
                                    "strides": None}
    return torch.as_tensor(_Arr(), device="cuda")


def test_cfg1_full_range_sample_vs_oracle_and_rule_check():
    """configs[1] at full size on the default lane-resident launch (148 CTAs, 3-lane groups,
    partial last group), checked over the WHOLE lane range:
    * a seeded random sample of 4,096 pairs spread over all 2^20 lanes (plus the first and last
      lane of every CTA's first group, the CTA-stride boundary and the partial last group):
      XOR and AND ciphertexts equal the oracle's compact NAND chain on host-encrypted inputs
      (each pair's generator position reached by PCG64 jump-ahead: independent of device
      encryption);
    * every one of the 2^21 output ciphertexts is identical with the instantiation that waits
      on every in-group producer (dbg bit 21) -- the check of the compiled-out RAW waits rule
      (tc_nand_resident.cuh slot table);
    * every output decrypts to the right bit."""
    import torch
    from oracle import gsw
    lanes = 1 << 20
    scheme = GswScheme(DEFAULT_PARAMS)
    keys = scheme.keygen(1)
    rng = np.random.default_rng(1)
    bits = rng.integers(0, 2, (lanes, 2))
    enc_state = rng.bit_generator.state                  # generator position of pair 0's a
    eng = GpuEngine(scheme, keys=keys, rng=rng, batch_size=lanes, device_encrypt=True)
    a, b = eng.input_block(bits)
    x, y = xor_(a, b), and_(a, b)
    prog = eng.flush()
    assert eng.last_compile["schedule"] == "resident" and prog.launches == 1
    got = eng.read_back_bits([x, y])
    assert (got[0] == (bits[:, 0] ^ bits[:, 1])).all()
    assert (got[1] == (bits[:, 0] & bits[:, 1])).all()
    # sample: random lanes + structural boundaries of the resident launch
    n_groups, grid = -(-lanes // 3), 148
    special = [0, 1, 2, 3 * grid - 1, 3 * grid, 3 * grid + 1, lanes - 2, lanes - 1]
    special += [3 * c for c in range(grid)] + [3 * c + 2 for c in range(grid)]
    smp = np.unique(np.concatenate([np.random.default_rng(2024).choice(lanes, 4096, replace=False),
                                    np.array(special)]))
    vx, vy = (eng.read_nodes([h.node], [0], lanes=smp)[0] for h in (x, y))
    p = gsw.DEFAULT
    step = p.n_ct * p.m // 2                              # raw 64-bit draws per ciphertext
    gen = np.random.Generator(np.random.PCG64())
    bad = []
    for i, lane in enumerate(smp.tolist()):
        ins = []
        for j in (0, 1):
            gen.bit_generator.state = enc_state
            gen.bit_generator.advance((2 * lane + j) * step)
            ins.append(scheme.encrypt_many(keys.public_key, [int(bits[lane, j])], gen)[0].astype(np.int64))
        va, vb = ins
        n1 = gsw.hom_nand_compact(p, va, vb)
        t1 = gsw.hom_nand_compact(p, n1, va)              # n1 is noisier: swapped left
        t2 = gsw.hom_nand_compact(p, n1, vb)
        want_x = gsw.hom_nand_compact(p, t1, t2)
        want_y = gsw.hom_nand_compact(p, n1, n1)
        if not (np.array_equal(vx[i], want_x) and np.array_equal(vy[i], want_y)):
            bad.append(lane)
    assert not bad, f"{len(bad)} sampled pairs differ from the oracle, first lanes {bad[:8]}"
    # the compiled-out waits: same outputs with every in-group producer awaited
    ctx = eng.ctx
    sx, sy = (eng._slot[h.node] * lanes for h in (x, y))
    ref = [_store_view(ctx, s0, lanes).clone() for s0 in (sx, sy)]
    ctx.set_debug(1 << 21)
    prog.run(lanes)
    ctx.sync()
    ctx.set_debug(0)
    torch.cuda.synchronize()
    for r, s0 in zip(ref, (sx, sy)):
        assert torch.equal(r, _store_view(ctx, s0, lanes))
    del ref
    torch.cuda.empty_cache()


def test_tiled_program_refuses_level_fallback():
    """A tiled program has no level structure: if the dataflow kernel cannot run (SIMT kernel
    forced) it must fail loudly rather than run its dependent ops as one level."""
    from paper_1611_08769_b200 import DeviceError, _native
    scheme = GswScheme(DEFAULT_PARAMS)
    keys = scheme.keygen(1)
    eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(1), batch_size=2048,
                    device_encrypt=True, schedule="tiled")
    a, b = eng.input_block(np.random.default_rng(2).integers(0, 2, (2048, 2)))
    x = xor_(a, b)
    prog = eng.flush()
    scheme.ctx.set_kernel(_native.KERNEL_SIMT)
    with pytest.raises(DeviceError, match="dataflow"):
        prog.run(2048)
    scheme.ctx.set_kernel(_native.KERNEL_AUTO)


@pytest.mark.parametrize("lanes", [4096, 4097])
def test_resident_schedule_equals_levels_bit_exact(lanes):
    """schedule='resident': XOR + AND per lane in one lane-resident launch (inputs loaded once,
    intermediates in shared memory) -- every output ciphertext equals the level schedule's, with
    and without operand reuse between a lane's consecutive gates, also with a lane count that
    leaves the last 3-lane group partial."""
    scheme = GswScheme(DEFAULT_PARAMS)
    keys = scheme.keygen(1)
    bits = np.random.default_rng(9).integers(0, 2, (lanes, 2))
    outs = {}
    for variant in ("levels", "resident", "resident-noreuse"):
        schedule = variant.split("-")[0]
        eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(1), batch_size=lanes,
                        device_encrypt=True, schedule=schedule)
        eng.ctx.set_debug(1 << 20 if variant == "resident-noreuse" else 0)   # bit 20: no operand reuse
        a, b = eng.input_block(bits)
        x, y = xor_(a, b), and_(a, b)
        prog = eng.flush()
        if schedule == "resident":
            assert prog.launches == 1                      # partial last lane group included
        outs[variant] = eng.node_values([x, y])
        assert (eng.read_back_bits([x, y]) == np.stack([bits[:, 0] ^ bits[:, 1], bits[:, 0] & bits[:, 1]])).all()
        prog.run(lanes)                                    # re-running rewrites identical values
        assert np.array_equal(eng.node_values([x, y]), outs[variant])
        eng.ctx.set_debug(0)
    assert np.array_equal(outs["levels"], outs["resident"])
    assert np.array_equal(outs["levels"], outs["resident-noreuse"])


def test_resident_random_small_programs_equal_levels():
    """Random programs of <= 8 gates over 512 lanes (complemented operands, reused temporaries,
    outputs also read later): lane-resident launches equal level launches ciphertext for
    ciphertext."""
    from paper_1611_08769_b200.gates import nor_, not_, or_, xnor_
    scheme = GswScheme(DEFAULT0_PARAMS)
    keys = scheme.keygen(2)
    rng = np.random.default_rng(12)
    gates = [not_, and_, or_, xor_, nor_, xnor_]
    checked = 0
    for trial in range(12):
        plan = [(int(rng.integers(0, len(gates))), int(rng.integers(0, 50)), int(rng.integers(0, 50)))
                for _ in range(int(rng.integers(1, 4)))]
        bits = rng.integers(0, 2, (512, int(rng.integers(1, 4))))
        res = {}
        for schedule in ("levels", "resident"):
            eng = GpuEngine(scheme, keys=keys, rng=np.random.default_rng(3), batch_size=512,
                            device_encrypt=True, schedule=schedule)
            pool = eng.input_block(bits)
            for g, i, j in plan:
                p1, p2 = pool[i % len(pool)], pool[j % len(pool)]
                pool.append(gates[g](p1) if gates[g] is not_ else gates[g](p1, p2))
            keep = [h for h in pool[len(bits[0]):] if not h.const][-3:]
            prog = eng.flush()
            if prog is None or not keep:
                break
            res[schedule] = (eng.node_values(keep), prog.launches)
        if len(res) == 2:
            assert np.array_equal(res["levels"][0], res["resident"][0])
            checked += res["resident"][1] == 1
    assert checked >= 4


def test_flow_schedule_falls_back_outside_its_range():
    """schedule='flow' over 2 lanes keeps the program's level launches (the warp-dataflow launch
    serves one lane); at the default geometry the C ABI refuses the mode and says why."""
    from paper_1611_08769_b200.errors import DeviceError
    pname, seed, (F, f), dims, _ = FFT_CONFIGS["cfg0"]
    scheme = GswScheme(EXACT_PARAMS)
    keys = scheme.keygen(seed)
    rng, vals = config_signal("cfg0")
    eng = GpuEngine(scheme, keys=keys, batch_size=2, lane_rngs=[np.random.default_rng(7), np.random.default_rng(8)],
                    device_encrypt=True, schedule="flow")
    out = fft_1d(input_signal(eng, np.stack([vals, vals[::-1]]), FixedFormat(F, f)))
    got = read_signal_ints(eng, out)
    assert eng.last_compile["schedule"] == "flow"
    want = model_outputs("cfg0", np.stack([vals, vals[::-1]]))
    assert np.array_equal(got, want)
    # default geometry: fhegpu_prog_set_flow is unsupported, loudly
    s2 = GswScheme(DEFAULT0_PARAMS)
    k2 = s2.keygen(1)
    e2 = GpuEngine(s2, keys=k2, rng=np.random.default_rng(1), schedule="flow")
    a, b = e2.input_bit(1), e2.input_bit(0)
    with pytest.raises(DeviceError, match="k = 3, ell = 17"):
        e2.read_back(xor_(a, b))
