// C ABI of RLM-sort (recurse-last multiway mergesort, rlm.py:86-132) on one
// GPU: SURVEY §8(f) row 4.
//
// Elements are (key, origin tag) pairs, the tag being the element's index in
// the PE-major input — the reference's (key, origin_pe, origin_pos) order
// (core.py:19-43).  Every PE array is kept sorted by (key, tag):
//   1. local sort of every PE (rlm.py:96-97);
//   2. per level and group: exact cut positions for the r equal parts
//      (_cut_points rlm.py:53-83) by device multisequence selection
//      (k_rlm.cu), pieces copied into the delivery's member arrays (the
//      same C++ planners as AMS-sort's deliver, delivery.py:151-455), then
//      every member re-sorted by (key, tag) — the merge of its received
//      sorted runs (merge_runs rlm.py:48-50, 113-115);
//   3. level reports (rlm.py:118-131).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "ctx.h"

namespace {

constexpr uint64_t kRlmCopyItem = 8192;  // keys per k_copy_ranges work item

void push_items(std::vector<uint64_t>& items, uint64_t s0, uint64_t d0, uint64_t len) {
  for (uint64_t o = 0; o < len; o += kRlmCopyItem) {
    items.push_back(s0 + o);
    items.push_back(d0 + o);
    items.push_back(std::min<uint64_t>(kRlmCopyItem, len - o));
  }
}

int copy_items(ams_ctx* c, const std::vector<uint64_t>& items, const void* sk, const void* sv, void* dk,
               void* dv, uint64_t n) {
  if (items.empty()) return AMS_OK;
  Stage& sc = c->st_copy;
  sc.reset();
  const size_t oi = sc.put(items);
  AMS_CK(sc.upload(c->stream));
  AMS_CK(launch_copy_ranges(c->stream, sc.dev<uint64_t>(oi), (int)(items.size() / 3), sk, dk, sv, dv, n));
  c->launches += 1;
  return AMS_OK;
}

// Sort every segment of (K, T) by (key, tag): by tag first, then stably by
// key.  (K, T) -> (X, Y) -> (K2, T2); tmp buffers are scratch.
int sort_by_key_tag(ams_ctx* c, void* K, void* T, void* X, void* Y, void* K2, void* T2, void* tmpa,
                    void* tmpb, int nseg, const uint64_t* off, const uint64_t* len, uint64_t n,
                    const std::vector<uint64_t>& klo, const std::vector<uint64_t>& khi, bool tags_sorted) {
  int rc;
  void* sk = K;
  void* st = T;
  if (!tags_sorted) {
    std::vector<uint64_t> tlo(nseg, 0), thi(nseg, n ? n - 1 : 0);
    // keys = tags, values = keys -> (Y = sorted tags, X = their keys)
    if ((rc = sort_segments_lohi(c, T, K, tmpa, tmpb, Y, X, AMS_KEY_U64, nseg, off, len, tlo, thi))) return rc;
    sk = X;
    st = Y;
  }
  return sort_segments_lohi(c, sk, st, tmpa, tmpb, K2, T2, AMS_KEY_U64, nseg, off, len, klo, khi);
}

}  // namespace

extern "C" {

int ams_rlm_sort_run(ams_ctx_t* c, int levels, const int32_t* group_counts, int scheme,
                     int64_t master_seed, const char* stream_id, int key_kind, int p,
                     const uint64_t* pe_sizes, const void* keys, const void* vals, void* out,
                     void* out_origin, void* out_vals, uint64_t* out_pe_sizes,
                     ams_rlm_report_t* reports) {
  if (!c || !group_counts || !pe_sizes || !stream_id) return set_error(AMS_EINVAL, "null argument");
  // LevelPlan.__post_init__ (rlm.py:29-41).
  if (p < 1) return set_error(AMS_EINVAL, "need at least one PE");
  std::string gc = "(";
  for (int lv = 0; lv < levels; ++lv) gc += std::to_string(group_counts[lv]) + (levels == 1 ? "," : lv + 1 < levels ? ", " : "");
  gc += ")";
  {
    int remaining = p;
    for (int lv = 0; lv < levels; ++lv) {
      const int r = group_counts[lv];
      if (r < 1 || remaining % r != 0)
        return set_error(AMS_EINVAL, "group counts " + gc + " do not divide " + std::to_string(p));
      remaining /= r;
    }
    if (remaining != 1)
      return set_error(AMS_EINVAL, "group counts " + gc + " do not telescope " + std::to_string(p) + " to 1");
  }
  if (scheme < AMS_SCHEME_SIMPLE || scheme > AMS_SCHEME_RANDOMIZED)
    return set_error(AMS_EINVAL, "unknown delivery scheme");
  if (key_kind < AMS_KEY_U64 || key_kind > AMS_KEY_F64) return set_error(AMS_EINVAL, "unknown key kind");
  uint64_t n = 0;
  for (int i = 0; i < p; ++i) n += pe_sizes[i];
  if (n && (!keys || !out)) return set_error(AMS_EINVAL, "null key buffer");
  if (vals && !out_vals) return set_error(AMS_EINVAL, "values need an output buffer");
  if (n >= 0xFFFFFFFFull) return set_error(AMS_EINVAL, "input too large for this path");
  AMS_ON_DEVICE(c->device);
  std::vector<uint64_t> sizes(pe_sizes, pe_sizes + p);
  c->rlm_levels.assign(levels, ams_ctx::RlmLevel{});
  // Eight n-key buffers: current (A), simple layout (B), members (C), scratch (D).
  const size_t wb = 8 * ((size_t)std::max<uint64_t>(n, 1) + 2);
  void* buf[8];
  {
    DevBuf* all[8] = {&c->work[0], &c->work[1], &c->work_v[0], &c->work_v[1], &c->tags0,
                      &c->rlm_buf[0], &c->rlm_buf[1], &c->rlm_buf[2]};
    for (int i = 0; i < 8; ++i) {
      AMS_CK(all[i]->ensure(wb));
      buf[i] = all[i]->p;
    }
  }
  void *Ak = buf[0], *At = buf[1], *Bk = buf[2], *Bt = buf[3], *Ck = buf[4], *Ct = buf[5], *Dk = buf[6],
       *Dt = buf[7];
  std::vector<uint64_t> offs(p + 1, 0);
  for (int i = 0; i < p; ++i) offs[i + 1] = offs[i] + sizes[i];
  int rc;
  // 1. Local sort (rlm.py:96-97): keys order-mapped to u64, tags = input index.
  std::vector<uint64_t> klo(p, 0), khi(p, ~0ULL);
  if (n) {
    AMS_CK(launch_map_keys(c->stream, keys, Bk, n, key_kind, AMS_KEY_U64));
    AMS_CK(launch_iota(c->stream, Bt, n));
    c->launches += 2;
    if ((rc = sort_by_key_tag(c, Bk, Bt, nullptr, nullptr, Ak, At, Dk, Dt, p, offs.data(), sizes.data(), n,
                              klo, khi, true)))
      return rc;
  }
  // 2. Levels.
  std::vector<int32_t> gf{0}, gn{p};
  std::vector<uint64_t> glo{0}, ghi{~0ULL};  // key bounds of every group
  for (int lv = 0; lv < levels; ++lv) {
    const int r = group_counts[lv];
    const int G = (int)gf.size();
    for (int i = 0; i < p; ++i) offs[i + 1] = offs[i] + sizes[i];
    ams_ctx::RlmLevel& rec = c->rlm_levels[lv];
    rec.r = r;
    rec.group_first = gf;
    rec.group_npe = gn;
    rec.sizes_before = sizes;
    rec.cuts.assign((size_t)p * (r + 1), 0);
    rec.new_sizes.assign(p, 0);
    rec.stats.assign((size_t)G * 4, 0);
    // Queries: targets strictly inside (0, n_g) (rlm.py:60-68).
    std::vector<RlmQuery> qs;
    std::vector<int> q_group, q_part;
    std::vector<std::vector<uint64_t>> targets(G);
    uint64_t cut_words = 0;
    for (int g = 0; g < G; ++g) {
      uint64_t n_g = 0;
      for (int j = 0; j < gn[g]; ++j) n_g += sizes[gf[g] + j];
      const uint64_t part = n_g / r, rem = n_g % r;
      uint64_t acc = 0;
      for (int t = 0; t + 1 < r; ++t) {
        acc += part + ((uint64_t)t < rem ? 1 : 0);
        targets[g].push_back(acc);
        if (acc > 0 && acc < n_g) {
          qs.push_back(RlmQuery{gf[g], gn[g], acc, cut_words});
          q_group.push_back(g);
          q_part.push_back(t);
          cut_words += (uint64_t)gn[g];
        }
      }
    }
    std::vector<uint64_t> h_cuts(cut_words), h_skey(qs.size());
    if (!qs.empty()) {
      Stage& sr = c->st_rlm;
      sr.reset();
      const size_t oo = sr.put(offs), oq = sr.put(qs);
      AMS_CK(sr.upload(c->stream));
      AMS_CK(c->rlm_cuts.ensure(8 * (size_t)cut_words));
      AMS_CK(c->rlm_skey.ensure(8 * qs.size()));
      AMS_CK(launch_rlm_select(c->stream, static_cast<const uint64_t*>(Ak), static_cast<const uint64_t*>(At),
                               sr.dev<uint64_t>(oo), sr.dev<RlmQuery>(oq), (int)qs.size(), n ? n - 1 : 0,
                               c->rlm_cuts.as<uint64_t>(), c->rlm_skey.as<uint64_t>()));
      c->launches += 1;
      AMS_CK(cudaMemcpyAsync(h_cuts.data(), c->rlm_cuts.p, 8 * (size_t)cut_words, cudaMemcpyDeviceToHost,
                             c->stream));
      AMS_CK(cudaMemcpyAsync(h_skey.data(), c->rlm_skey.p, 8 * qs.size(), cudaMemcpyDeviceToHost, c->stream));
      AMS_CK(cudaStreamSynchronize(c->stream));
    }
    // Cut matrix (rlm.py:69-83) and the splitter key of every part boundary.
    std::vector<std::vector<uint64_t>> bkey(G);
    for (int g = 0; g < G; ++g) {
      bkey[g].assign(r + 1, 0);
      bkey[g][0] = glo[g];
      bkey[g][r] = ghi[g];
      uint64_t n_g = 0;
      for (int j = 0; j < gn[g]; ++j) n_g += sizes[gf[g] + j];
      for (int j = 0; j < gn[g]; ++j) {
        uint64_t* row = rec.cuts.data() + (size_t)(gf[g] + j) * (r + 1);
        row[r] = sizes[gf[g] + j];
        for (int t = 0; t + 1 < r; ++t)
          if (targets[g][t] >= n_g) row[t + 1] = sizes[gf[g] + j];  // == 0 stays 0
      }
      for (int t = 0; t + 1 < r; ++t) bkey[g][t + 1] = targets[g][t] == 0 ? glo[g] : ghi[g];
    }
    for (size_t q = 0; q < qs.size(); ++q) {
      const int g = q_group[q], t = q_part[q];
      for (int j = 0; j < gn[g]; ++j)
        rec.cuts[(size_t)(gf[g] + j) * (r + 1) + t + 1] = h_cuts[qs[q].out + j];
      bkey[g][t + 1] = h_skey[q];
    }
    // Pieces -> simple layout E (part-major, then source member) -> members.
    std::vector<uint64_t> items, items2, pieces, slices;
    bool relayout = false;
    for (int g = 0; g < G; ++g) {
      const int P = gn[g];
      const uint64_t gstart = offs[gf[g]];
      pieces.assign((size_t)P * r, 0);
      uint64_t at = gstart;
      for (int t = 0; t < r; ++t)
        for (int j = 0; j < P; ++j) {
          const uint64_t* row = rec.cuts.data() + (size_t)(gf[g] + j) * (r + 1);
          const uint64_t len = row[t + 1] - row[t];
          pieces[(size_t)j * r + t] = len;
          if (len) push_items(items, offs[gf[g] + j] + row[t], at, len);
          at += len;
        }
      uint64_t* ns = rec.new_sizes.data() + gf[g];
      uint64_t* st4 = rec.stats.data() + 4 * (size_t)g;
      if (scheme == AMS_SCHEME_SIMPLE) {
        if ((rc = ams_deliver_simple(P, r, pieces.data(), ns, st4))) return rc;
        continue;
      }
      const int cap = P * (2 * r + 2) + 16;
      slices.assign(3 * (size_t)cap, 0);
      int nsl = 0;
      const std::string ls = std::string(stream_id) + "/L" + std::to_string(lv) + "-g" + std::to_string(gf[g]);
      if (scheme == AMS_SCHEME_PERMUTED)
        rc = ams_deliver_permuted(P, r, master_seed, ls.c_str(), pieces.data(), ns, slices.data(), cap, &nsl, st4);
      else if (scheme == AMS_SCHEME_RANDOMIZED)
        rc = ams_deliver_randomized(P, r, master_seed, ls.c_str(), pieces.data(), ns, slices.data(), cap, &nsl,
                                    st4);
      else
        rc = ams_deliver_deterministic(P, r, gf[g], pieces.data(), ns, slices.data(), cap, &nsl, st4);
      if (rc) return rc;
      // One member per subgroup: the member array is the part itself
      // (receivers concatenate by source, simnet.py:324-325) — no relayout.
      if (P / r > 1) {
        relayout = true;
        for (int q = 0; q < nsl; ++q)
          push_items(items2, gstart + slices[3 * q], gstart + slices[3 * q + 1], slices[3 * q + 2]);
      }
    }
    if ((rc = copy_items(c, items, Ak, At, Bk, Bt, n))) return rc;
    void *Mk = Bk, *Mt = Bt, *Xk = Ck, *Xt = Ct;
    if (relayout) {
      // (all groups of a level have the same member count, so they relayout together)
      if ((rc = copy_items(c, items2, Bk, Bt, Ck, Ct, n))) return rc;
      Mk = Ck; Mt = Ct; Xk = Bk; Xt = Bt;
    }
    // Next level's groups and their key bounds; members re-sorted by (key, tag).
    std::vector<int32_t> nf, nn;
    std::vector<uint64_t> nlo, nhi;
    std::vector<uint64_t> mlo(p), mhi(p);
    for (int g = 0; g < G; ++g) {
      const int step = gn[g] / r;
      for (int t = 0; t < r; ++t) {
        nf.push_back(gf[g] + t * step);
        nn.push_back(step);
        nlo.push_back(bkey[g][t]);
        nhi.push_back(std::max(bkey[g][t], bkey[g][t + 1]));
        for (int m = 0; m < step; ++m) {
          mlo[gf[g] + t * step + m] = nlo.back();
          mhi[gf[g] + t * step + m] = nhi.back();
        }
      }
    }
    sizes = rec.new_sizes;
    for (int i = 0; i < p; ++i) offs[i + 1] = offs[i] + sizes[i];
    if (n && (rc = sort_by_key_tag(c, Mk, Mt, Xk, Xt, Ak, At, Dk, Dt, p, offs.data(), sizes.data(), n, mlo,
                                   mhi, false)))
      return rc;
    if (reports) {
      ams_rlm_report_t& rp = reports[lv];
      std::memset(&rp, 0, sizeof rp);
      rp.level = lv + 1;
      rp.r = r;
      rp.max_load = *std::max_element(sizes.begin(), sizes.end());
      rp.min_load = *std::min_element(sizes.begin(), sizes.end());
      for (int g = 0; g < G; ++g) {
        rp.max_words = std::max(rp.max_words, rec.stats[4 * g + 0]);
        rp.max_msgs = std::max(rp.max_msgs, rec.stats[4 * g + 1]);
        rp.max_sent_msgs = std::max(rp.max_sent_msgs, rec.stats[4 * g + 2]);
        rp.max_recv_msgs = std::max(rp.max_recv_msgs, rec.stats[4 * g + 3]);
      }
    }
    gf.swap(nf);
    gn.swap(nn);
    glo.swap(nlo);
    ghi.swap(nhi);
  }
  // 3. Outputs: keys back in the caller's type, origins, gathered payloads.
  if (n) {
    AMS_CK(launch_map_keys(c->stream, Ak, out, n, AMS_KEY_U64, key_kind));
    c->launches += 1;
    if (out_origin)
      AMS_CK(cudaMemcpyAsync(out_origin, At, 8 * (size_t)n, cudaMemcpyDeviceToDevice, c->stream));
    if (vals) {
      AMS_CK(launch_gather_vals(c->stream, vals, At, out_vals, n));
      c->launches += 1;
    }
  }
  if (out_pe_sizes) std::memcpy(out_pe_sizes, sizes.data(), sizeof(uint64_t) * p);
  return AMS_OK;
}

int ams_rlm_level_dims(ams_ctx_t* c, int level, int* r, int* ngroups, int* npe) {
  if (!c || level < 0 || level >= (int)c->rlm_levels.size()) return set_error(AMS_EINVAL, "no such RLM level");
  const ams_ctx::RlmLevel& L = c->rlm_levels[level];
  if (r) *r = L.r;
  if (ngroups) *ngroups = (int)L.group_first.size();
  if (npe) *npe = (int)L.new_sizes.size();
  return AMS_OK;
}

int ams_rlm_level(ams_ctx_t* c, int level, int32_t* group_first, int32_t* group_npe,
                  uint64_t* sizes_before, uint64_t* cuts, uint64_t* new_sizes, uint64_t* stats) {
  if (!c || level < 0 || level >= (int)c->rlm_levels.size()) return set_error(AMS_EINVAL, "no such RLM level");
  const ams_ctx::RlmLevel& L = c->rlm_levels[level];
  auto put = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
  };
  put(group_first, L.group_first);
  put(group_npe, L.group_npe);
  put(sizes_before, L.sizes_before);
  put(cuts, L.cuts);
  put(new_sizes, L.new_sizes);
  put(stats, L.stats);
  return AMS_OK;
}

}  // extern "C"
