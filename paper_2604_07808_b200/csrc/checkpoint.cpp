// checkpoint.cpp — grass_save_state / grass_load_state (SURVEY 8(f) f4,
// SPEC.md:192-199): self-describing header + per-layer blobs, 64-bit lengths,
// CRC32 (zlib); verify-then-apply.
#include <zlib.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "context.h"

namespace gapi {

// ---- checkpoint ------------------------------------------------------------
const char kCkMagic[8] = {'G', 'R', 'A', 'S', 'S', 'C', 'K', '1'};
const uint32_t kCkVersion = 3;  // 2: n_always in the header; 3: bf16 master flags + config fingerprint

uint32_t crc_update(uint32_t crc, const void* p, size_t n) {
  const Bytef* b = static_cast<const Bytef*>(p);
  while (n > 0) {
    const uInt k = (uInt)std::min<size_t>(n, 1u << 30);
    crc = (uint32_t)crc32(crc, b, k);
    b += k;
    n -= k;
  }
  return crc;
}

template <class T>
void put(std::vector<char>* h, const T* p, size_t n) {
  const char* b = reinterpret_cast<const char*>(p);
  h->insert(h->end(), b, b + sizeof(T) * n);
}

constexpr int kCkInts = 6;  // n_layers, world, rank, committed, dtype, n_always

// The hyperparameters a checkpoint's state depends on (a load into a context
// configured differently is rejected): Eq. 3/4 (tau, alpha, normalisation),
// AdamW (betas, eps, weight decay), the sampler (gamma, seed, policy) and the
// schedule (T_p, T_s, T_u).
struct CkFingerprint {
  double tau, alpha, beta1, beta2, eps, weight_decay;
  int32_t normalize_mgn, gamma, T_p, T_s, T_u, policy;
  uint64_t seed;
};
static_assert(sizeof(CkFingerprint) == 80, "fingerprint layout");
CkFingerprint ck_fingerprint(const grass_ctx* c) {
  CkFingerprint f;
  std::memset(&f, 0, sizeof(f));
  const grass_config& k = c->cfg;
  f.tau = k.tau;
  f.alpha = k.alpha;
  f.beta1 = k.beta1;
  f.beta2 = k.beta2;
  f.eps = k.eps;
  f.weight_decay = k.weight_decay;
  f.normalize_mgn = k.normalize_mgn;
  f.gamma = k.gamma;
  f.T_p = k.T_p;
  f.T_s = k.T_s;
  f.T_u = k.T_u;
  f.policy = k.policy;
  f.seed = k.seed;
  return f;
}

// mvalid: the bf16 master flags (DevState::mvalid, read from the device by
// the caller) — a master written by grass_write_master before any update
// (t = 0) is valid and must survive a save / load.
std::vector<char> ck_header(grass_ctx* c, const std::vector<int32_t>& mvalid) {
  std::vector<char> h;
  const int32_t ints[kCkInts] = {c->nl,         c->cfg.world,         c->cfg.rank, c->committed ? 1 : 0,
                                 c->cfg.param_dtype, c->cfg.n_always};
  put(&h, ints, kCkInts);
  const CkFingerprint fp = ck_fingerprint(c);
  put(&h, &fp, 1);
  put(&h, mvalid.data(), c->nl);
  put(&h, c->numel.data(), c->nl);
  put(&h, c->shard_len.data(), c->nl);
  put(&h, c->t.data(), c->nl);
  put(&h, c->mgn.data(), c->nl);
  put(&h, c->probs.data(), c->nl);
  put(&h, h_S(c), c->nl);
  put(&h, h_c(c), c->nl);
  return h;
}


}  // namespace gapi

using namespace gapi;

extern "C" {

grass_status grass_save_state(grass_ctx* c, const char* path) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!path) return c->fail(GRASS_E_INVALID, "path is NULL");
  grass_status s = drain(c, false);
  if (s == GRASS_OK) s = flush_cache(c);
  if (s != GRASS_OK) return s;
  // t_l lives on the device (it advances in captured graphs too)
  CUDA_TRY(c, cudaMemcpy(c->t.data(), c->st.t, sizeof(long long) * c->nl, cudaMemcpyDeviceToHost));
  std::vector<int32_t> mvalid(c->nl, 0);
  CUDA_TRY(c, cudaMemcpy(mvalid.data(), c->st.mvalid, sizeof(int32_t) * c->nl, cudaMemcpyDeviceToHost));
  const std::vector<char> hdr = ck_header(c, mvalid);
  FILE* f = std::fopen(path, "wb");
  if (!f) return c->fail(GRASS_E_IO, std::string("cannot open ") + path + " for writing");
  bool ok = true;
  const uint64_t hlen = hdr.size();
  const uint32_t hcrc = crc_update(0, hdr.data(), hdr.size());
  ok = ok && std::fwrite(kCkMagic, 1, 8, f) == 8;
  ok = ok && std::fwrite(&kCkVersion, 4, 1, f) == 1;
  ok = ok && std::fwrite(&hlen, 8, 1, f) == 1;
  ok = ok && std::fwrite(&hcrc, 4, 1, f) == 1;
  ok = ok && std::fwrite(hdr.data(), 1, hdr.size(), f) == hdr.size();
  std::vector<float> tmp;
  for (int l = 0; ok && l < c->nl; ++l) {
    // one blob per layer: m, v [, master] shards, fp32
    const size_t n = (size_t)c->shard_len[l];
    tmp.resize((size_t)c->ns * n);
    for (int a = 0; a < c->ns && s == GRASS_OK; ++a) s = copy_state_out(c, a, l, tmp.data() + a * n);
    if (s != GRASS_OK) {
      std::fclose(f);
      return s;
    }
    const uint64_t len = 4 * (uint64_t)tmp.size();
    const uint32_t crc = crc_update(0, tmp.data(), len);
    ok = ok && std::fwrite(&len, 8, 1, f) == 1 && std::fwrite(&crc, 4, 1, f) == 1;
    ok = ok && std::fwrite(tmp.data(), 4, tmp.size(), f) == tmp.size();
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return c->fail(GRASS_E_IO, std::string("short write to ") + path);
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

grass_status grass_load_state(grass_ctx* c, const char* path) try {
  if (!c) return set_thread_err(GRASS_E_INVALID, "ctx is NULL");
  if (!path) return c->fail(GRASS_E_INVALID, "path is NULL");
  grass_status s = drain(c, false);
  if (s != GRASS_OK) return s;
  FILE* f = std::fopen(path, "rb");
  if (!f) return c->fail(GRASS_E_IO, std::string("cannot open ") + path);
  auto bad = [&](grass_status st, const std::string& m) {
    std::fclose(f);
    return c->fail(st, m);
  };
  char magic[8];
  uint32_t ver = 0, hcrc = 0;
  uint64_t hlen = 0;
  if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kCkMagic, 8) != 0)
    return bad(GRASS_E_IO, "not a GRASS checkpoint (bad magic)");
  if (std::fread(&ver, 4, 1, f) != 1 || ver != kCkVersion) return bad(GRASS_E_IO, "unsupported version");
  if (std::fread(&hlen, 8, 1, f) != 1 || std::fread(&hcrc, 4, 1, f) != 1) return bad(GRASS_E_IO, "truncated header");
  const int nl = c->nl;
  const size_t want = 4 * kCkInts + sizeof(CkFingerprint) + (size_t)nl * (4 + 3 * 8 + 4 * 8);
  if (hlen != want) return bad(GRASS_E_INVALID, "checkpoint was written for a different layer count");
  std::vector<char> hdr(hlen);
  if (std::fread(hdr.data(), 1, hlen, f) != hlen) return bad(GRASS_E_IO, "truncated header");
  if (crc_update(0, hdr.data(), hlen) != hcrc) return bad(GRASS_E_IO, "header CRC32 mismatch (integrity error)");
  const char* p = hdr.data();
  auto take = [&](void* dst, size_t k) {
    std::memcpy(dst, p, k);
    p += k;
  };
  int32_t ints[kCkInts];
  take(ints, sizeof(ints));
  CkFingerprint fp;
  take(&fp, sizeof(fp));
  std::vector<int32_t> mvalid(nl);
  take(mvalid.data(), 4 * nl);
  std::vector<int64_t> numel(nl), slen(nl), t(nl);
  std::vector<double> mgn(nl), probs(nl), S(nl);
  std::vector<long long> cnt(nl);
  take(numel.data(), 8 * nl);
  take(slen.data(), 8 * nl);
  take(t.data(), 8 * nl);
  take(mgn.data(), 8 * nl);
  take(probs.data(), 8 * nl);
  take(S.data(), 8 * nl);
  take(cnt.data(), 8 * nl);
  if (ints[0] != nl || ints[1] != c->cfg.world || ints[2] != c->cfg.rank || ints[4] != c->cfg.param_dtype ||
      ints[5] != c->cfg.n_always || numel != c->numel || slen != c->shard_len)
    return bad(GRASS_E_INVALID,
               "checkpoint does not match this context (N_L, n_always, N_p, dtype, world or rank)");
  const CkFingerprint mine = ck_fingerprint(c);
  if (std::memcmp(&fp, &mine, sizeof(fp)) != 0)
    return bad(GRASS_E_INVALID, "checkpoint was written by a context with other hyperparameters (tau, alpha, "
                                "normalisation, betas, eps, weight decay, gamma, seed, policy or T_p/T_s/T_u)");
  const long blobs = std::ftell(f);
  // pass 1: verify every blob's length and CRC32 before touching the context
  std::vector<char> buf(64u << 20);
  for (int l = 0; l < nl; ++l) {
    uint64_t len = 0;
    uint32_t crc = 0;
    if (std::fread(&len, 8, 1, f) != 1 || std::fread(&crc, 4, 1, f) != 1)
      return bad(GRASS_E_IO, "truncated layer blob header");
    if (len != 4 * (uint64_t)c->ns * (uint64_t)slen[l])
      return bad(GRASS_E_IO, "corrupt layer blob length (integrity error)");
    uint32_t got = 0;
    for (uint64_t done = 0; done < len;) {
      const size_t k = (size_t)std::min<uint64_t>(buf.size(), len - done);
      if (std::fread(buf.data(), 1, k, f) != k) return bad(GRASS_E_IO, "truncated layer blob");
      got = crc_update(got, buf.data(), k);
      done += k;
    }
    if (got != crc) return bad(GRASS_E_IO, "layer " + std::to_string(l) + " CRC32 mismatch (integrity error)");
  }
  // pass 2: apply (cached copies are superseded by the checkpoint)
  std::fseek(f, blobs, SEEK_SET);
  if (c->cache_slots) {
    for (int k = 0; k < c->cache_slots; ++k) {
      c->slot_layer[k] = -1;
      c->slot_dirty[k] = 0;
    }
    std::fill(c->layer_slot.begin(), c->layer_slot.end(), -1);
  }
  std::vector<float> tmp;
  for (int l = 0; l < nl; ++l) {
    std::fseek(f, 12, SEEK_CUR);
    const size_t n = (size_t)slen[l];
    tmp.resize((size_t)c->ns * n);
    if (std::fread(tmp.data(), 4, tmp.size(), f) != tmp.size()) return bad(GRASS_E_IO, "read failed");
    for (int a = 0; a < c->ns; ++a) {
      if ((s = copy_state_in(c, a, l, tmp.data() + a * n)) != GRASS_OK) {
        std::fclose(f);
        return s;
      }
    }
    if (c->bf16) c->master_valid[l] = mvalid[l] ? 1 : 0;
  }
  std::fclose(f);
  c->t = t;
  CUDA_TRY(c, cudaMemcpy(c->st.t, t.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice));
  if (c->bf16) {
    std::vector<int> mv(nl);
    for (int l = 0; l < nl; ++l) mv[l] = c->master_valid[l];
    CUDA_TRY(c, cudaMemcpy(c->st.mvalid, mv.data(), sizeof(int) * nl, cudaMemcpyHostToDevice));
  }
  c->mgn = mgn;
  c->probs = probs;
  c->committed = ints[3] != 0;
  std::vector<char> blk(16 * (size_t)nl);
  std::memcpy(blk.data(), S.data(), 8 * (size_t)nl);
  std::memcpy(blk.data() + 8 * (size_t)nl, cnt.data(), 8 * (size_t)nl);
  CUDA_TRY(c, cudaMemcpy(c->d_mgn, blk.data(), blk.size(), cudaMemcpyHostToDevice));
  return GRASS_OK;
} catch (...) {
  return api_exception(c);
}

}  // extern "C"
