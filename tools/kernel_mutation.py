"""Mutation check of the GPU parity tests: each mutant is a copy of
paper_2604_07808_b200/csrc/ with ONE plausible kernel mistake patched in (a
text replacement below), built into its own libgrass; a fast subset of the GPU
tests must FAIL for every one of them.  The product source carries no mutation
hooks: the mistakes exist only in the patched copies under build/msrc/.

    python tools/kernel_mutation.py build      # here (nvcc cross-compiles)
    python tools/kernel_mutation.py run        # on the GPU box
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CSRC = os.path.join(ROOT, "paper_2604_07808_b200", "csrc")
OUTDIR = os.path.join(ROOT, "build", "mutants")
SRCDIR = os.path.join(ROOT, "build", "msrc")
K = "kernels.cu"
S = "stream_kernel.cuh"
OFF = "offload.cpp"
HOT = "hot_path.cpp"
CK = "checkpoint.cpp"

# k: (what, [(file, product text, mutated text), ...]) — every product text
# must occur in the file (all occurrences are replaced)
MUTANTS = {
    1: ("AdamW: weight decay dropped",
        [(K, "const float t1 = th * s.decay;", "const float t1 = th;")]),
    2: ("AdamW: bias correction 1/sqrt(1-b2^t) dropped",
        [(K, "const float den = fmaf(sq, s.inv_bc2s, s.eps);", "const float den = fmaf(sq, 1.0f, s.eps);")]),
    3: ("norm: one warp's partial left out of each tile sum",
        [(S, "for (int w = 0; w < kConsumerWarps; ++w) p += red[i & 1][tid][w];",
          "for (int w = 0; w < kConsumerWarps - 1; ++w) p += red[i & 1][tid][w];")]),
    4: ("ragged tail: last element of a segment skipped",
        [(S, "if (e + j < ne) {", "if (e + j < ne - 1) {")]),
    5: ("DP: gradient not scaled by 1/W",
        [(S, "const float gs = b.gscale;", "const float gs = 1.0f;")]),
    6: ("DP: last rank's gradient slice not summed",
        [(S, "gacc[k0][q].x += x.x; gacc[k0][q].y += x.y; gacc[k0][q].z += x.z; gacc[k0][q].w += x.w;",
          "if (r != b.npeer - 1) { gacc[k0][q].x += x.x; gacc[k0][q].y += x.y; gacc[k0][q].z += x.z; gacc[k0][q].w += x.w; }")]),
    7: ("bf16: parameter copy truncated instead of RNE",
        [(S, "__device__ __forceinline__ uint32_t f2bf(float f) {",
          "__device__ __forceinline__ uint32_t f2bf(float f) {\n  return __float_as_uint(f) >> 16;")]),
    8: ("step prologue: t_l not advanced (bias corrections of step 1 forever)",
        [(K, "  st.t[l] = t;\n", "\n")]),
    9: ("P2P: theta' not stored into the last rank's parameters",
        [(S, "for (int q = 0; q < ntp; ++q) {", "for (int q = 0; q < ntp - 1; ++q) {")]),
    10: ("bf16: master never initialised from the bf16 parameter",
         [(S, "const bool init = BF16 && UPDATE && (DEVB ? dinit[s] : st.init_now[sg.layer]);",
           "const bool init = false;")]),
    11: ("non-finite norm not flagged",
         [(K, "atomicMax(st.flag, INT_MAX - layer);  // smallest id wins", "(void)0;")]),
    12: ("norm: all-tiles warp reduction (warp_sum_perm) fed in tile order instead of the lane's permuted order",
         [(S, "const int pm = (!UPDATE && ne == kUnit) ? (lane >> MS::SHIFT) & (GS - 1) : 0;", "const int pm = 0;")]),
    16: ("bf16 K1 fast path: the stage handed back even when a sum left fp32's range (fallback re-reads a refilled stage)",
         [(S, "          if (__all_sync(0xffffffffu, ok)) {", "          if (true) {")]),
    13: ("bf16 norm: the last square of each thread's fp32 8-square sum dropped",
         [(S, "      s = __fmaf_rn(w, w, s);", "      s = __fmaf_rn(w, 0.f, s);")]),
    15: ("bf16 norm: the fp32 8-square sum used even where it underflows (no exact fallback)",
         [(S, "  return __float_as_uint(s) - 0x0D800000u <= 0x7F7FFFFFu - 0x0D800000u;", "  return true;")]),
    17: ("offload: a chunk's fetch does not wait for the ring slot's previous write-back",
         [(OFF, "    if (overlap && c->slot_used[slot]) CUDA_TRY(c, cudaStreamWaitEvent(sh, c->ev_free[slot], 0));\n", "")]),
    18: ("offload: a layer's fetch does not wait for its previous step's write-back",
         [(OFF, "  if (overlap && c->layer_done_valid[l])  // previous write-back of this layer\n"
                "    CUDA_TRY(c, cudaStreamWaitEvent(c->h2d, c->ev_layer_done[l], 0));\n", "")]),
    19: ("period residency: a victim's write-back does not wait for the updates before it",
         [(HOT, "    if (c->cfg.overlap && (s = wait_pending(c, c->d2h)) != GRASS_OK) return s;\n", "")]),
    20: ("device schedule: Eq. 4 EMA weights swapped (alpha on the old MGN)",
         [(K, "sM[l] = committed ? a.alpha * w + (1.0 - a.alpha) * sM[l] : w;",
           "sM[l] = committed ? (1.0 - a.alpha) * w + a.alpha * sM[l] : w;")]),
    21: ("device schedule: sampler mass R not renormalised over the still-available layers (R6)",
         [(K, "      const double R = c;",
           "      double R = 0.0;\n      for (int j = 0; j < ns; ++j) R += sP[j];")]),
    22: ("device schedule: the sampling period not advanced",
         [(K, "const uint64_t period = a.period == ~0ull ? s_pctr + 1 : a.period;",
           "const uint64_t period = a.period == ~0ull ? s_pctr : a.period;")]),
    23: ("device step: K3 does not advance t_l (the step prologue's state update)",
         [(K, "      st.t[layer] += 1;\n", "\n")]),
    24: ("device step: K2's inline prologue takes t_l instead of t_l + 1",
         [(S, "const long long t = st.t[l] + 1;\n      const double lr = b.dev_lr_ptr",
           "const long long t = st.t[l];\n      const double lr = b.dev_lr_ptr")]),
    25: ("device step: the fused commit's done counter not reset (no commit after the first step)",
         [(K, "if (threadIdx.x == 0) *fa.done_ctr = 0;", "(void)0;")]),
    26: ("device schedule: the commit ignores the non-finite flag (commits a window missing the layer)",
         [(K, "      if (s_flag != 0) s_err = 2;", "      if (false) s_err = 2;")]),
    27: ("clipping: the update ignores the clip coefficient (R17)",
         [(S, "const float cf = (UPDATE && b.coef) ? *b.coef : 1.0f;", "const float cf = 1.0f;")]),
    28: ("clipping: coefficient without min(1, .) (small gradients scaled up)",
         [(K, "coef[0] = (float)fmin(1.0, a.max_norm / (sqrt(tot) + 1e-6));",
           "coef[0] = (float)(a.max_norm / (sqrt(tot) + 1e-6));")]),
    29: ("checkpoint: a load into a context with other hyperparameters accepted (fingerprint not checked)",
         [(CK, "if (std::memcmp(&fp, &mine, sizeof(fp)) != 0)", "if (false)")]),
    30: ("checkpoint: t_l restored on the host only (the device step counts keep their old values)",
         [(CK, "  CUDA_TRY(c, cudaMemcpy(c->st.t, t.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice));\n", "")]),
    14: ("P2P barrier self-test: start barrier removed",
         [(K, "    a.which = 0;  // start barrier: every rank has read its rows of this round\n"
              "    const int n_save = a.n;\n    a.n = 0;\n    p2p_sync_cta(a);\n    a.n = n_save;\n", "")]),
}
TESTS = ("test_step_layers_vs_oracle_multi_step or test_norms_ragged_sizes_vs_oracle or "
         "test_bf16_mixed_precision_vs_oracle or test_p2p_virtual_ranks_vs_oracle or "
         "test_zero_grad_zero_state_is_identity_on_theta or test_nonfinite_gradient_reported_and_not_recorded or "
         "test_norms_probe_equals_update_bitwise or test_norms_integer_grads_exact_bf16 or "
         "test_p2p_barrier_protocol_selftest or test_bf16_norms_tiny_and_huge_gradients or "
         "test_norms_all_tiles_reduction_keeps_each_tile_apart or test_offload_pipeline_happens_before_under_stress or "
         "test_device_schedule_equals_host_schedule or test_device_schedule_commit_and_sampler_against_oracle or "
         "test_device_schedule_policies_equal_host or test_device_schedule_nonfinite_gradient_stops_commits_and_is_reported or "
         "test_clipping_vs_oracle or test_checkpoint_roundtrip_and_integrity or "
         "test_checkpoint_keeps_written_master_and_rejects_other_hyperparameters")


def patched_source(k: int) -> str:
    """A copy of csrc/ with mutant k's replacements applied (fails loudly if a
    product text is missing, so the patch set cannot silently go stale)."""
    d = os.path.join(SRCDIR, f"m{k}")
    shutil.rmtree(d, ignore_errors=True)
    shutil.copytree(CSRC, d)
    for fname, old, new in MUTANTS[k][1]:
        p = os.path.join(d, fname)
        s = open(p).read()
        if old not in s:
            raise SystemExit(f"mutant {k}: product text not found in {fname}: {old!r}")
        open(p, "w").write(s.replace(old, new))
    return d


def build(only=()):
    from paper_2604_07808_b200 import build as b
    os.makedirs(OUTDIR, exist_ok=True)
    for k in (only or MUTANTS):
        b.build(force=True, src_dir=patched_source(k), out=os.path.join(OUTDIR, f"libgrass_m{k}.so"))
        print("built mutant", k, flush=True)


def _subset(lib):
    env = dict(os.environ)
    if lib:
        env["GRASS_LIB_PATH"] = lib
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                           "tests/test_gpu_parity.py", "tests/test_gpu_p2p.py", "tests/test_gpu_race.py",
                           "tests/test_gpu_device_schedule.py",
                           "-k", TESTS],
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)


def run(only=()):
    res = {}
    r = _subset(None)                      # control: the product library passes the subset
    res["product"] = {"passed": r.returncode == 0, "summary": (r.stdout.strip().splitlines() or [""])[-1]}
    print("product", res["product"], flush=True)
    for k, (what, _) in MUTANTS.items():
        if only and k not in only:
            continue
        r = _subset(os.path.join(OUTDIR, f"libgrass_m{k}.so"))
        failed = [l for l in r.stdout.splitlines() if l.startswith("FAILED")]
        res[k] = {"mutation": what, "killed": r.returncode != 0, "by": failed[:1]}
        print(k, res[k], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "kernel_mutation" + ("_subset" if only else "") + ".json"), "w") as f:
        json.dump(res, f, indent=1)
    muts = [v for k, v in res.items() if k != "product"]
    killed = sum(v["killed"] for v in muts)
    print(f"{killed}/{len(muts)} kernel mutations killed by the GPU parity tests; product passes: "
          f"{res['product']['passed']}")
    return 0 if killed == len(muts) and res["product"]["passed"] else 1


if __name__ == "__main__":
    if sys.argv[1:] == ["check"]:  # CPU: every patch still applies to the product source
        for k in MUTANTS:
            patched_source(k)
        print(f"{len(MUTANTS)} mutant patches apply")
        sys.exit(0)
    if sys.argv[1:2] == ["build"]:
        sys.exit(build([int(x) for x in sys.argv[2:]]))
    sys.exit(run([int(x) for x in sys.argv[2:]]))
