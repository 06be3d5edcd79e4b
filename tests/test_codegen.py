"""CPU: the generic lowered-term -> CUDA compiler generates sources that NVRTC
compiles for sm_100a (no GPU needed), for every program in the corpus, and
whose host-compiled form (codegen.cpu_source, g++ -ffp-contract=off: the same
fp32 operations in the same order) matches the reference interpreter."""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from paper_2002_02268_b200 import binomial, codegen, schedules
from paper_2002_02268_b200._ref import S

CHAIN = """
def chain = fun(x : 8.f32 => x |> map(fun(a => add(a)(a))) |> map(fun(b => mult(b)(b))) |> map(fun(c => add(c)(1.0))));
"""
# a reduce whose array accumulator is read transposed: not elementwise, so
# the compiler switches to destination passing (one thread per batch entry)
TRACC = """
def tracc = fun(x : 5.4.3.3.f32 => fun(y : 3.3.f32 => x |> mapSeq(fun(b => b |> reduceSeq(fun(acc => fun(m =>
  zip(transpose(acc))(m) |> mapSeq(fun(p => zip(fst(p))(snd(p)) |> mapSeq(fun(q => add(fst(q))(snd(q)))))))))(y)))));
"""
MM_BT = """
def mmbt = fun(a : 6.5.f32 => fun(bt : 7.5.f32 =>
  a |> map(fun(r => bt |> map(fun(c => dot(r, c)))))));
"""


def corpus():
    s = S()
    out = {"mm_highlevel": schedules.mm(8, 12, 16), "chain": s.ir.parse(CHAIN),
           "mm_bt": s.ir.parse(MM_BT), "tracc": s.ir.parse(TRACC)}
    for n in schedules.SCHEDULE_NAMES:
        out[n] = schedules.apply(n, 64, 32, 16).term
    for n in binomial.SCHEDULE_NAMES:
        out["bf_" + n] = binomial.apply(n, 5, 9)
    # a user schedule the templates do not know: tile(16,16) without reorder
    st, nf, tv, rules = s.strategy, s.normal_forms, s.traversals, s.rules
    user = st.seq(nf.dfnf_seq(tv.top_down(schedules.tile(16, 16)),
                              tv.top_down(st.seq(tv.is_reduce, rules.make_split(2)))), nf.LOWER_TO_C)
    out["user_tile16"] = st.run_strategy(user, schedules.mm(32, 48, 8))[0].term
    return out


@pytest.mark.parametrize("name,term", list(corpus().items()))
def test_generated_source_compiles(name, term):
    pytest.importorskip("cuda.bindings.nvrtc")
    c = codegen.compile_term(term)
    assert "elv_generated" in c.source
    cubin = codegen.nvrtc_cubin(c)
    assert len(cubin) > 1000


def test_shapes_and_errors():
    s = S()
    c = codegen.compile_term(schedules.apply("blocking", 64, 32, 16).term)
    assert c.in_shapes == ((64, 16), (16, 32)) and c.out_shape == (64, 32)
    bad = s.ir.parse("def f = fun(a : 4.f32 => zip(a)(a));")          # result is pairs
    with pytest.raises(codegen.CodegenError):
        codegen.compile_term(bad)
    illtyped = schedules.apply("blocking", 64, 64, 1031).term
    with pytest.raises(codegen.CodegenError):
        codegen.compile_term(illtyped)


def _cpu_run(c, args, tmp_path):
    src, so = tmp_path / "k.cpp", tmp_path / "k.so"
    src.write_text(codegen.cpu_source(c))
    subprocess.run(["g++", "-O1", "-ffp-contract=off", "-shared", "-fPIC", "-o", str(so), str(src)], check=True)
    lib = ctypes.CDLL(str(so))
    out = np.zeros(c.out_shape, np.float32)
    arr = (ctypes.c_void_p * len(args))(*[a.ctypes.data for a in args])
    lib.elv_run_cpu(arr, out.ctypes.data_as(ctypes.c_void_p), ctypes.c_longlong(c.threads))
    return out


@pytest.mark.parametrize("name,term", list(corpus().items()))
def test_generated_code_matches_reference_interpreter(name, term, tmp_path):
    """Code generation checked on the host: every program in the corpus
    (the seven GEMM schedules, the four binomial schedules, a user tiling,
    a non-elementwise reduce) against stratir.interp.run (checker only)."""
    from paper_2002_02268_b200 import synth
    s = S()
    c = codegen.compile_term(term)
    args = [synth.matrix(*shp, 3, i) if len(shp) == 2 else
            synth.uniform(int(np.prod(shp)), 3, i).reshape(shp) for i, shp in enumerate(c.in_shapes)]
    got = _cpu_run(c, args, tmp_path)
    ref = np.array(s.interp.run(term, [a.tolist() for a in args]), np.float64)
    assert got.shape == ref.shape
    assert np.all(np.abs(got - ref) <= 64 * 4 * 2.0 ** -23), name


def test_thread_mappings():
    """Lifted (elementwise) array reduces become per-element scalar folds --
    one thread per output scalar, no per-thread accumulator arrays; a
    non-elementwise accumulator switches to destination passing."""
    for n in schedules.SCHEDULE_NAMES:
        c = codegen.compile_term(schedules.apply(n, 64, 32, 16).term)
        assert c.mode == "per-scalar" and c.threads == 64 * 32 and "accbuf" not in c.source, n
    c = codegen.compile_term(S().ir.parse(TRACC))
    assert c.mode == "destination-passing" and c.threads == 5 and "accbuf" in c.source


def test_vector_program_is_not_taken_for_a_gemm():
    """CPU half of the generic-fallback check: the template path rejects a
    two-vector program with the "no B200 kernel" prefix that sends interp.run
    to the generated-kernel path (not the reference's matrix map error)."""
    from paper_2002_02268_b200 import interp
    term = S().ir.parse("""
def vadd = fun(a : 4.f32 => fun(b : 4.f32 => zip(a)(b) |> map(fun(p => add(fst(p))(snd(p))))));
""")
    with pytest.raises(S().interp.EvalError) as err:
        interp._run_template(term, [[1.0, 2.0, 3.0, 4.0], [1.0, 1.0, 1.0, 1.0]])
    assert interp._no_template(err.value)


@pytest.mark.parametrize("name", ["user_tile16", "blocking", "parallel", "baseline", "cacheBlocks"])
def test_register_tile_mode_is_bitwise_the_per_scalar_code(name, tmp_path, monkeypatch):
    """Mode A' (a 4x4 / 2x2 register tile of outputs per thread) replicates
    the per-scalar statements per output with private locals: every output
    keeps the per-scalar operation sequence, so the host-compiled results are
    bitwise those of the per-scalar kernel (and match the interpreter)."""
    from paper_2002_02268_b200 import synth
    term = corpus()[name]
    monkeypatch.setattr(codegen, "MIN_TILE_THREADS", 10 ** 9)
    plain = codegen.compile_term(term)
    monkeypatch.setattr(codegen, "MIN_TILE_THREADS", 1)
    tiled = codegen.compile_term(term)
    assert plain.mode == "per-scalar" and tiled.mode.startswith("register-tile"), (plain.mode, tiled.mode)
    args = [synth.matrix(*shp, 4, i) for i, shp in enumerate(plain.in_shapes)]
    a = _cpu_run(plain, args, tmp_path / "a" if (tmp_path / "a").mkdir() is None else tmp_path)
    b = _cpu_run(tiled, args, tmp_path / "b" if (tmp_path / "b").mkdir() is None else tmp_path)
    np.testing.assert_array_equal(a, b)
    ref = np.array(S().interp.run(term, [x.tolist() for x in args]), np.float64)
    assert np.all(np.abs(b - ref) <= 64 * 4 * 2.0 ** -23)


def test_smem_tile_mode_source_and_host_guard(monkeypatch):
    """A contraction of at least 256 x 256 outputs compiles in the shared-memory
    tile mode (GPU-only: staged chunks, __syncthreads, f32x2-paired fmaf); the
    host emulation refuses it, and with the mode off the same term falls back
    to the register-tile mode (what the host tests compile)."""
    from paper_2002_02268_b200._ref import S
    s = S()
    st, nf, tv, rules = s.strategy, s.normal_forms, s.traversals, s.rules
    strat = st.seq(nf.dfnf_seq(tv.top_down(schedules.tile(16, 16)),
                               tv.top_down(st.seq(tv.is_reduce, rules.make_split(2)))), nf.LOWER_TO_C)
    term = st.run_strategy(strat, schedules.mm(256, 256, 64))[0].term
    c = codegen.compile_term(term)
    assert c.mode.startswith("smem-tile") and c.grid == (4, 4) and c.block == 128
    assert "__syncthreads" in c.source and "fma.rn.f32x2" in c.source and "elv_fma2(" in c.source
    with pytest.raises(codegen.CodegenError):
        codegen.cpu_source(c)
    monkeypatch.setattr(codegen, "SMEM_TILE", False)
    c2 = codegen.compile_term(term)
    assert c2.mode.startswith("register-tile") and not c2.grid
    # outputs below the threshold, or not multiples of 64, never use it
    monkeypatch.setattr(codegen, "SMEM_TILE", True)
    small = st.run_strategy(strat, schedules.mm(64, 64, 64))[0].term
    assert not codegen.compile_term(small).mode.startswith("smem-tile")


def test_gemmcall_launch_counts():
    """GemmCall.count_launches: the library's launches per call (the bench's
    gpu_launches claim), by variant and problem size."""
    from types import SimpleNamespace as P
    from paper_2002_02268_b200.interp import GemmCall
    assert GemmCall.count_launches(P(variant=0, M=64, N=64, K=64)) == 1
    assert GemmCall.count_launches(P(variant=6, M=4096, N=4096, K=4096)) == 2          # packs + GEMM
    assert GemmCall.count_launches(P(variant=7, M=1024, N=1024, K=1024)) == 3          # zero + split + GEMM (fix-up inside)
    assert GemmCall.count_launches(P(variant=7, M=32768, N=32768, K=8192)) == 4        # + separate fix-up
    assert GemmCall.count_launches(P(variant=8, M=32768, N=32768, K=8192)) == 5        # 3 prepare + GEMM + fix-up
    assert GemmCall.count_launches(P(variant=8, M=1024, N=1024, K=256)) == 3           # K < 512 runs as 7
    assert GemmCall.count_launches(P(variant=8, M=2048, N=2048, K=2048)) == 5          # mid-size: pair kernel


def test_pair_kernel_choice_model():
    """interp.pair_kernel (the library's pair / 1-CTA choice): the 1-CTA
    kernel for the paper's 1024^3 and for 1536^3 (measured faster there), the
    cta_group::2 kernel from 2048^3 up (profiles/r2/small/mid_pair.jsonl) and
    whenever there are at least as many pair tiles as SMs."""
    from paper_2002_02268_b200.interp import pair_kernel
    assert not pair_kernel(1024, 1024) and not pair_kernel(1536, 1536) and not pair_kernel(1000, 1031)
    assert not pair_kernel(4096, 256)
    assert pair_kernel(2048, 2048) and pair_kernel(3072, 3072) and pair_kernel(2560, 2560)
    assert pair_kernel(32768, 32768) and pair_kernel(4096 * 4, 2048)
