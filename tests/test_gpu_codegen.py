"""GPU: generated kernels (codegen.py) against the reference interpreter
itself (stratir.interp.run from baseline/_ref, used here only as a checker),
and the template kernels against the generated ones."""

import numpy as np
import pytest
import torch

import oracle
from paper_2002_02268_b200 import binomial, codegen, interp, schedules, synth
from paper_2002_02268_b200._ref import S

from test_codegen import corpus

pytestmark = pytest.mark.gpu


def _inputs(term, seed=3):
    c = codegen.compile_term(term)
    return [synth.matrix(*shp, seed, i) if len(shp) == 2 else
            synth.uniform(int(np.prod(shp)), seed, i).reshape(shp) for i, shp in enumerate(c.in_shapes)]


@pytest.mark.parametrize("name,term", list(corpus().items()))
def test_generated_kernel_matches_reference_interpreter(cuda, name, term):
    s = S()
    args = _inputs(term)
    ref = np.array(s.interp.run(term, [a.tolist() for a in args]), np.float64)
    got = codegen.run(term, [torch.from_numpy(a).to(cuda) for a in args]).cpu().numpy().astype(np.float64)
    assert got.shape == ref.shape
    # fp32 with separately rounded ops (--fmad=false) vs the interpreter's
    # f64: every program here folds at most 64 terms of magnitude <= 4
    assert np.all(np.abs(got - ref) <= 64 * 4 * 2.0 ** -23), name


def test_run_falls_back_to_generated_kernel(cuda):
    """interp.run: a schedule the templates do not know still runs (on the GPU)."""
    term = corpus()["user_tile16"]
    A = synth.matrix(32, 8, 1, 0)
    B = synth.matrix(8, 48, 1, 1)
    C = interp.run(term, [A, B])
    ok, worst = oracle.check(C, oracle.mm_f64(A, B), oracle.absprod_np(A, B), 8)
    assert ok, worst


@pytest.mark.parametrize("name", schedules.SCHEDULE_NAMES)
def test_template_and_generated_kernels_agree(cuda, name):
    M, N, K = 64, 96, 64
    term = schedules.apply(name, M, N, K).term
    A = torch.from_numpy(synth.matrix(M, K, 2, 0)).to(cuda)
    B = torch.from_numpy(synth.matrix(K, N, 2, 1)).to(cuda)
    gen = codegen.run(term, [A, B]).cpu().numpy()
    tpl = interp.run_tensor(term, A, B).cpu().numpy()
    Ah, Bh = A.cpu().numpy(), B.cpu().numpy()
    ref, ab = oracle.mm_interp_f64(Ah, Bh, name), oracle.absprod_np(Ah, Bh)
    assert oracle.check(gen, ref, ab, K)[0] and oracle.check(tpl, ref, ab, K)[0]
    # both fold each output as one fmaf chain in k order: the same bits
    np.testing.assert_array_equal(gen, tpl)


@pytest.mark.parametrize("name", ["parallel", "loopPerm"])
def test_tiled_generated_kernel_at_1024(cuda, name):
    """The generated kernel at 1024^3 (shared-memory tile mode: a contraction)
    is bitwise the template kernel's result (same fmaf chain per output)."""
    n = 1024
    term = schedules.apply(name, n, n, n).term
    assert codegen.kernel_for(term).c.mode.startswith("smem-tile")
    A = torch.empty((n, n), device=cuda); synth.fill_device(A, 3, 0)
    B = torch.empty((n, n), device=cuda); synth.fill_device(B, 3, 1)
    assert torch.equal(codegen.run(term, [A, B]), interp.run_tensor(term, A, B))


def _user_terms(M, N=None, K=None):
    N, K = N or M, K or M
    from paper_2002_02268_b200._ref import S
    st, nf, tv, rules = S().strategy, S().normal_forms, S().traversals, S().rules
    out = {}
    for name, (ti, tj, sp) in {"tile16_split2": (16, 16, 2), "tile32x64_split8": (32, 64, 8),
                               "tile64_split4": (64, 64, 4)}.items():
        strat = st.seq(nf.dfnf_seq(tv.top_down(schedules.tile(ti, tj)),
                                   tv.top_down(st.seq(tv.is_reduce, rules.make_split(sp)))), nf.LOWER_TO_C)
        out[name] = st.run_strategy(strat, schedules.mm(M, N, K))[0].term
    return out


@pytest.mark.parametrize("shape", [(256, 256, 256), (1024, 1024, 1024), (512, 256, 768), (256, 1024, 128)],
                         ids=lambda s: "x".join(map(str, s)))
def test_smem_tile_mode_is_bitwise_the_register_tile_mode(cuda, shape, monkeypatch):
    """Mode A'' stages each load site's values in shared memory and keeps every
    output's per-scalar statement sequence: the same bits as the register-tile
    (and per-scalar) kernels, for user schedules outside the templates and the
    seven schedules."""
    M, N, K = shape
    terms = _user_terms(M, N, K)
    terms.update({name: schedules.apply(name, M, N, K).term for name in ("blocking", "cacheBlocks", "baseline")})
    A = torch.empty((M, K), device=cuda); synth.fill_device(A, 7, 0)
    B = torch.empty((K, N), device=cuda); synth.fill_device(B, 7, 1)
    stream = torch.cuda.current_stream().cuda_stream
    for name, term in terms.items():
        outs = {}
        for smem in (True, False):
            monkeypatch.setattr(codegen, "SMEM_TILE", smem)
            k = codegen.Kernel(codegen.compile_term(term))
            assert k.c.mode.startswith("smem-tile") == smem, (name, k.c.mode)
            C = torch.empty((M, N), device=cuda)
            k([A, B], C, stream)
            outs[smem] = C
        torch.cuda.synchronize()
        assert torch.equal(outs[True], outs[False]), name
    ref = A.double() @ B.double()
    assert (outs[True].double() - ref).abs().max().item() < 1e-3


VEC_ADD = """
def vadd = fun(a : 4.f32 => fun(b : 4.f32 => zip(a)(b) |> map(fun(p => add(fst(p))(snd(p))))));
"""


def test_two_vector_arguments_reach_the_generic_compiler(cuda):
    """A two-argument program over vectors is no GEMM schedule: interp.run
    must not stop at the matrix-operand check but compile it,
    like the reference evaluates it (interp.py:157-162)."""
    s = S()
    term = s.ir.parse(VEC_ADD)
    a, b = [1.0, 2.0, 3.0, 4.0], [1.0, 1.0, 1.0, 1.0]
    assert s.interp.run(term, [a, b]) == [2.0, 3.0, 4.0, 5.0]
    assert interp.run(term, [a, b]) == [2.0, 3.0, 4.0, 5.0]
