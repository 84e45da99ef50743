// Single-process multi-device driver (SURVEY §8(b) "one host thread drives
// all GPUs", §8(e)): one context per device, level 1 across the devices by
// peer pointers, the later levels and the final sort as ams_sort_run
// continuations on every device.
//
//   PE i lives on device i * G / p; group_counts[0] % G == 0, so every
//   level-1 group lands on one device and nothing after level 1 crosses
//   devices.  Level 1 (ams.py:214-268 for the group of all PEs):
//     draw           once on the host (draw_sample, ams.py:157-175)
//     sample         every device gathers its share and copies it into the
//                    other devices' sample buffers (the all-gather of
//                    fastsort.py:84-93)
//     splitters      replicated on every device (identical)
//     classify       local PEs; the host joins the histograms (the allreduce
//                    of ams.py:236-237) and the key range
//     plan           once on the host (optimal_group_plan, ams.py:238)
//     scatter        every device stores its pieces straight into the owner
//                    devices' receive buffers (ams_level_scatter_peers), at
//                    the offsets of Network.exchange (simnet.py:294-335)
//     delivery       non-simple schemes: the members of a subgroup share a
//                    device, so the relayout of the simple layout is local
//   Blocking per-device steps run on one host thread per device.
//
// Several contexts may share one physical device (devices[] may repeat):
// the same code path, used by the single-GPU tests.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "ctx.h"

struct ams_mg {
  std::vector<ams_ctx_t*> ctx;
  std::vector<cudaStream_t> streams;
  std::vector<int> devices;
  // level-1 records of the last run
  int r = 0, p = 0, nb = 0, nb_stride = 0;
  uint64_t drawn = 0;
  std::vector<uint32_t> hist;
  std::vector<uint64_t> sizes_before, boundaries, loads, new_sizes, stats;
  uint64_t max_load = 0;
};

namespace {

// Runs f(i) for every device on its own host thread; the first error wins.
template <class F>
int for_devices(int G, F f) {
  std::vector<int> rc(G, AMS_OK);
  std::vector<std::string> msg(G);
  if (G == 1) {
    rc[0] = f(0);
    return rc[0];
  }
  std::vector<std::thread> th;
  for (int i = 0; i < G; ++i)
    th.emplace_back([&, i] {
      rc[i] = f(i);
      if (rc[i]) msg[i] = ams_last_error();
    });
  for (auto& t : th) t.join();
  for (int i = 0; i < G; ++i)
    if (rc[i]) return set_error(rc[i], msg[i]);
  return AMS_OK;
}

int sync_all(ams_mg* m) {
  for (size_t i = 0; i < m->ctx.size(); ++i) {
    DeviceGuard dg(m->devices[i]);
    AMS_CK(cudaStreamSynchronize(m->streams[i]));
  }
  return AMS_OK;
}

}  // namespace

extern "C" {

int ams_mg_create(const int* devices, int ngpu, ams_mg_t** out) {
  if (!devices || !out || ngpu < 1 || ngpu > 64) return set_error(AMS_EINVAL, "bad device list");
  ams_mg* m = new ams_mg();
  for (int i = 0; i < ngpu; ++i) {
    ams_ctx_t* c = nullptr;
    cudaStream_t st = nullptr;
    int rc = AMS_OK;
    {
      DeviceGuard dg(devices[i]);
      if (dg.err != cudaSuccess || cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
        rc = set_error(AMS_ECUDA, "cannot create a stream on device " + std::to_string(devices[i]));
    }
    if (!rc) rc = ams_ctx_create(devices[i], st, &c);
    if (rc) {
      ams_mg_destroy(m);
      return rc;
    }
    m->ctx.push_back(c);
    m->streams.push_back(st);
    m->devices.push_back(devices[i]);
  }
  // Peer access between distinct devices (stores into the owners' buffers).
  for (int i = 0; i < ngpu; ++i)
    for (int j = 0; j < ngpu; ++j) {
      if (devices[i] == devices[j]) continue;
      DeviceGuard dg(devices[i]);
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devices[i], devices[j]);
      if (!can) {
        ams_mg_destroy(m);
        return set_error(AMS_ECUDA, "no peer access between devices " + std::to_string(devices[i]) +
                                        " and " + std::to_string(devices[j]));
      }
      const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        ams_mg_destroy(m);
        return set_error(AMS_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
      }
      cudaGetLastError();
    }
  *out = m;
  return AMS_OK;
}

int ams_mg_destroy(ams_mg_t* m) {
  if (!m) return AMS_OK;
  for (size_t i = 0; i < m->ctx.size(); ++i) {
    ams_ctx_destroy(m->ctx[i]);
    DeviceGuard dg(m->devices[i]);
    cudaStreamDestroy(m->streams[i]);
  }
  delete m;
  return AMS_OK;
}

int ams_mg_size(const ams_mg_t* m) { return m ? (int)m->ctx.size() : 0; }

int ams_mg_ctx(ams_mg_t* m, int i, ams_ctx_t** out) {
  if (!m || !out || i < 0 || i >= (int)m->ctx.size()) return set_error(AMS_EINVAL, "no such context");
  *out = m->ctx[i];
  return AMS_OK;
}

int ams_mg_sort_run(ams_mg_t* m, const ams_params_t* prm, int p, const uint64_t* pe_sizes,
                    const void* const* keys, const void* const* vals, void* const* out,
                    void* const* out_vals, uint64_t* out_pe_sizes, ams_level_report_t* reports) {
  if (!m || !prm || !pe_sizes || !keys || !out) return set_error(AMS_EINVAL, "null argument");
  const int G = (int)m->ctx.size();
  const int k = prm->levels;
  if (k < 1 || k > AMS_MAX_LEVELS) return set_error(AMS_EINVAL, "levels outside 1..AMS_MAX_LEVELS");
  if (prm->level_base || prm->pe_base || prm->init_groups > 1)
    return set_error(AMS_EINVAL, "the multi-device driver runs whole sorts");
  uint64_t prod = 1;
  for (int lv = 0; lv < k; ++lv) {
    if (prm->group_counts[lv] < 1) return set_error(AMS_EINVAL, "group counts must be positive");
    prod *= (uint64_t)prm->group_counts[lv];
  }
  if (prm->overpartition < 1) return set_error(AMS_EINVAL, "overpartitioning factor must be at least 1");
  if (!(prm->imbalance > 0)) return set_error(AMS_EINVAL, "imbalance budget must be positive");
  if (p < 1 || prod != (uint64_t)p)
    return set_error(AMS_EINVAL, "group counts do not telescope " + std::to_string(p) + " PEs");
  const int r = prm->group_counts[0];
  if (p % G || r % G)
    return set_error(AMS_EINVAL, "first-level group count " + std::to_string(r) + " must be a multiple of the " +
                                     std::to_string(G) + " devices");
  if (!prm->stream_id) return set_error(AMS_EINVAL, "null argument");
  if (prm->scheme < AMS_SCHEME_SIMPLE || prm->scheme > AMS_SCHEME_RANDOMIZED)
    return set_error(AMS_EINVAL, "unknown delivery scheme");
  const bool det = prm->scheme != AMS_SCHEME_SIMPLE;
  if (det && vals)
    return set_error(AMS_EINVAL, "payloads are carried under the simple delivery scheme only");
  if (vals && !out_vals) return set_error(AMS_EINVAL, "values need an output buffer");
  const int pl = p / G, gpr = r / G, step = p / r;
  std::vector<uint64_t> sizes(pe_sizes, pe_sizes + p), offs(p + 1, 0);
  for (int i = 0; i < p; ++i) offs[i + 1] = offs[i] + sizes[i];
  const uint64_t n = offs[p];
  std::vector<uint64_t> rank_off(G + 1);
  for (int i = 0; i <= G; ++i) rank_off[i] = offs[(size_t)i * pl];
  for (int i = 0; i < G; ++i)
    if (rank_off[i + 1] > rank_off[i] && (!keys[i] || !out[i])) return set_error(AMS_EINVAL, "null key buffer");
  const double a = prm->oversampling > 0 ? prm->oversampling
                                         : 1.6 * std::log10((double)std::max<uint64_t>(n, 10));
  const double eps_l = std::pow(1.0 + prm->imbalance, 1.0 / k) - 1.0;
  int rc;
  // ---- draw (ams.py:224-228, 157-175) --------------------------------
  const uint64_t br0 = std::min<uint64_t>((uint64_t)prm->overpartition * r, n + 1);
  const uint64_t target = std::min<uint64_t>(n, std::max<uint64_t>(br0 - 1, (uint64_t)std::ceil(a * (double)br0)));
  std::vector<uint64_t> idx(std::max<uint64_t>(target, 1)), gpos(std::max<uint64_t>(target, 1));
  uint64_t drawn = 0;
  {
    const int32_t gf0 = 0, gn0 = p;
    if ((rc = ams_draw_sample_positions(prm->master_seed, prm->stream_id, 0, 1, &gf0, &gn0, &target,
                                        sizes.data(), offs.data(), target, idx.data(), gpos.data(), &drawn)))
      return rc;
  }
  const uint64_t S = drawn;
  const int nb = (int)std::min<uint64_t>(br0, S + 1);
  if (nb > AMS_MAX_BUCKETS)
    return set_error(AMS_EINVAL, std::to_string(nb) + " buckets exceed the supported " +
                                     std::to_string(AMS_MAX_BUCKETS));
  // share of every device: idx ascends (PE-major draw), so shares are contiguous
  std::vector<uint64_t> sh(G + 1, 0);
  for (int i = 0; i < G; ++i)
    sh[i + 1] = (uint64_t)(std::lower_bound(idx.begin(), idx.begin() + S, rank_off[i + 1]) - idx.begin());
  // ---- sample gather + exchange ------------------------------------------
  for (int i = 0; i < G; ++i) {
    ams_ctx* c = m->ctx[i];
    DeviceGuard dg(m->devices[i]);
    AMS_CK(c->s_keys.ensure(8 * std::max<uint64_t>(S, 1)));
    AMS_CK(c->s_pos.ensure(4 * std::max<uint64_t>(S, 1)));
  }
  std::vector<cudaEvent_t> ev(G, nullptr);
  for (int i = 0; i < G; ++i) {
    ams_ctx* c = m->ctx[i];
    const uint64_t cnt = sh[i + 1] - sh[i];
    std::vector<uint64_t> lidx(idx.begin() + sh[i], idx.begin() + sh[i + 1]);
    for (uint64_t& x : lidx) x -= rank_off[i];
    if (cnt && (rc = ams_level_sample(c, keys[i], prm->key_kind, cnt, lidx.data(), gpos.data() + sh[i],
                                      c->s_keys.as<uint64_t>() + sh[i], c->s_pos.as<uint32_t>() + sh[i])))
      return rc;
    DeviceGuard dg(m->devices[i]);
    for (int j = 0; j < G && cnt; ++j) {
      if (j == i) continue;
      ams_ctx* d = m->ctx[j];
      AMS_CK(cudaMemcpyAsync(d->s_keys.as<uint64_t>() + sh[i], c->s_keys.as<uint64_t>() + sh[i], 8 * cnt,
                             cudaMemcpyDefault, m->streams[i]));
      AMS_CK(cudaMemcpyAsync(d->s_pos.as<uint32_t>() + sh[i], c->s_pos.as<uint32_t>() + sh[i], 4 * cnt,
                             cudaMemcpyDefault, m->streams[i]));
    }
    AMS_CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    AMS_CK(cudaEventRecord(ev[i], m->streams[i]));
  }
  for (int i = 0; i < G; ++i) {
    DeviceGuard dg(m->devices[i]);
    for (int j = 0; j < G; ++j)
      if (j != i) AMS_CK(cudaStreamWaitEvent(m->streams[i], ev[j], 0));
  }
  // ---- splitters (replicated) and classification ------------------------
  const uint64_t soff[2] = {0, S};
  const int32_t nb32 = nb;
  const int nb_stride = nb;
  std::vector<uint32_t> hist((size_t)p * nb_stride, 0);
  rc = for_devices(G, [&](int i) -> int {
    ams_ctx* c = m->ctx[i];
    int e = ams_level_splitters(c, 1, c->s_keys.as<uint64_t>(), c->s_pos.as<uint32_t>(), soff, &nb32);
    if (e) return e;
    std::vector<uint64_t> loffs(pl), lsz(pl);
    std::vector<int32_t> sg(pl, 0);
    for (int j = 0; j < pl; ++j) {
      lsz[j] = sizes[(size_t)i * pl + j];
      loffs[j] = offs[(size_t)i * pl + j] - rank_off[i];
    }
    const int64_t posbase = (int64_t)rank_off[i];
    return ams_level_classify(c, keys[i], prm->key_kind, pl, loffs.data(), lsz.data(), sg.data(), 1, &posbase,
                              nb_stride, 1, 1, hist.data() + (size_t)i * pl * nb_stride);
  });
  for (int i = 0; i < G; ++i)
    if (ev[i]) cudaEventDestroy(ev[i]);
  if (rc) return rc;
  // key range of the whole input on every device
  {
    uint64_t lo = ~0ULL, hi = 0;
    for (int i = 0; i < G; ++i) {
      uint64_t mm[2];
      if ((rc = ams_get_minmax(m->ctx[i], mm))) return rc;
      if (rank_off[i + 1] > rank_off[i]) { lo = std::min(lo, mm[0]); hi = std::max(hi, mm[1]); }
    }
    if (n) {
      const uint64_t mm[2] = {lo, hi};
      for (int i = 0; i < G; ++i)
        if ((rc = ams_set_minmax(m->ctx[i], mm))) return rc;
    }
  }
  // ---- plan (replicated in the reference; once here) ---------------------
  m->r = r; m->p = p; m->nb = nb; m->nb_stride = nb_stride; m->drawn = S;
  m->sizes_before = sizes;
  m->boundaries.assign(r + 1, 0);
  m->loads.assign(r, 0);
  m->new_sizes.assign(p, 0);
  m->stats.assign(4, 0);
  {
    const int32_t gn0 = p;
    if ((rc = ams_plan_level(1, &gn0, &nb32, r, hist.data(), nb_stride, m->boundaries.data(), m->loads.data(),
                             &m->max_load, m->new_sizes.data(), m->stats.data())))
      return rc;
  }
  const std::vector<uint64_t>& bnd = m->boundaries;
  // pieces[j][g], group totals, owners and starts in the owners' buffers
  std::vector<uint64_t> pieces((size_t)p * r, 0), m_g(r, 0), g_start(r, 0), need(G, 0);
  for (int j = 0; j < p; ++j)
    for (int g = 0; g < r; ++g) {
      uint64_t s = 0;
      for (uint64_t b = bnd[g]; b < bnd[g + 1]; ++b) s += hist[(size_t)j * nb_stride + b];
      pieces[(size_t)j * r + g] = s;
      m_g[g] += s;
    }
  for (int d = 0; d < G; ++d) {
    uint64_t at = 0;
    for (int g = d * gpr; g < (d + 1) * gpr; ++g) { g_start[g] = at; at += m_g[g]; }
    need[d] = at;
  }
  std::vector<int32_t> owner(nb_stride, 0);
  for (int g = 0; g < r; ++g)
    for (uint64_t b = bnd[g]; b < bnd[g + 1]; ++b) owner[b] = g / gpr;
  // delivery of the scheme (member sizes, stats, relayout slices)
  std::vector<uint64_t> slices;
  int nsl = 0;
  if (det && n) {
    const int cap = p * (2 * r + 2) + 16;
    slices.assign(3 * (size_t)cap, 0);
    const std::string ls = std::string(prm->stream_id) + "/L0-g0";
    if (prm->scheme == AMS_SCHEME_PERMUTED)
      rc = ams_deliver_permuted(p, r, prm->master_seed, ls.c_str(), pieces.data(), m->new_sizes.data(),
                                slices.data(), cap, &nsl, m->stats.data());
    else if (prm->scheme == AMS_SCHEME_RANDOMIZED)
      rc = ams_deliver_randomized(p, r, prm->master_seed, ls.c_str(), pieces.data(), m->new_sizes.data(),
                                  slices.data(), cap, &nsl, m->stats.data());
    else
      rc = ams_deliver_deterministic(p, r, 0, pieces.data(), m->new_sizes.data(), slices.data(), cap, &nsl,
                                     m->stats.data());
    if (rc) return rc;
  }
  m->hist = hist;
  // ---- receive buffers, tags, scatter into the owners --------------------
  const bool with_v = vals != nullptr || det;
  std::vector<void*> dk(G), dv(G, nullptr);
  for (int i = 0; i < G; ++i) {
    ams_ctx* c = m->ctx[i];
    DeviceGuard dg(m->devices[i]);
    AMS_CK(c->peer_buf[0].ensure(8 * (need[i] + 2)));
    dk[i] = c->peer_buf[0].p;
    if (with_v) {
      AMS_CK(c->peer_buf[1].ensure(8 * (need[i] + 2)));
      dv[i] = c->peer_buf[1].p;
    }
    if (det) {
      const uint64_t nl = rank_off[i + 1] - rank_off[i];
      AMS_CK(c->rlm_buf[0].ensure(8 * std::max<uint64_t>(nl, 1)));
      if ((rc = ams_fill_iota(c, c->rlm_buf[0].p, nl, rank_off[i]))) return rc;
    }
  }
  // Receivers may still read their buffers (a previous sort's later levels).
  if ((rc = sync_all(m))) return rc;
  for (int i = 0; i < G; ++i) {
    ams_ctx* c = m->ctx[i];
    // cell base of every (local source PE, bucket) run in the (g, j, b) order
    std::vector<uint64_t> cb((size_t)pl * nb_stride, 0);
    for (int g = 0; g < r; ++g) {
      uint64_t before = 0;  // pieces of earlier source PEs for group g
      for (int j = 0; j < (i + 1) * pl; ++j) {
        if (j >= i * pl) {
          uint64_t within = 0;
          for (uint64_t b = bnd[g]; b < bnd[g + 1]; ++b) {
            cb[(size_t)(j - i * pl) * nb_stride + b] = g_start[g] + before + within;
            within += hist[(size_t)j * nb_stride + b];
          }
        }
        before += pieces[(size_t)j * r + g];
      }
    }
    // (a device without input still runs the step: it leaves the key
    // bounds of the device's groups in the context)
    const bool empty = rank_off[i + 1] == rank_off[i];
    const void* sk = empty ? dk[i] : keys[i];
    const void* sv = !with_v ? nullptr : empty ? dv[i] : det ? c->rlm_buf[0].p : vals[i];
    if ((rc = ams_level_scatter_peers(c, sk, sv, prm->key_kind, G, dk.data(), with_v ? dv.data() : nullptr,
                                      owner.data(), cb.data(), r, bnd.data(), i * gpr, gpr)))
      return rc;
  }
  if ((rc = sync_all(m))) return rc;  // every piece has landed
  // ---- non-simple delivery: local relayout of the simple layout ---------
  std::vector<const void*> src_k(G), src_v(G, nullptr);
  for (int i = 0; i < G; ++i) { src_k[i] = dk[i]; src_v[i] = dv[i]; }
  if (det && step > 1 && n) {
    for (int i = 0; i < G; ++i) {
      ams_ctx* c = m->ctx[i];
      uint64_t e0 = 0, d0 = 0;
      for (int g = 0; g < i * gpr; ++g) e0 += m_g[g];
      for (int j = 0; j < i * pl; ++j) d0 += m->new_sizes[j];
      std::vector<uint64_t> loc;
      for (int q = 0; q < nsl; ++q) {
        const uint64_t s0 = slices[3 * q], len = slices[3 * q + 2];
        if (len == 0 || s0 < e0 || s0 >= e0 + need[i]) continue;
        loc.push_back(s0 - e0);
        loc.push_back(slices[3 * q + 1] - d0);
        loc.push_back(len);
      }
      {
        DeviceGuard dg(m->devices[i]);
        AMS_CK(c->rlm_buf[1].ensure(8 * (need[i] + 2)));
        AMS_CK(c->rlm_buf[2].ensure(8 * (need[i] + 2)));
      }
      if ((rc = ams_copy_ranges(c, loc.data(), (int)(loc.size() / 3), dk[i], c->rlm_buf[1].p, dv[i],
                                c->rlm_buf[2].p)))
        return rc;
      src_k[i] = c->rlm_buf[1].p;
      src_v[i] = c->rlm_buf[2].p;
    }
  }
  // ---- level-1 report (ams.py:258-268, 294-308) -------------------------------
  if (reports) {
    ams_level_report_t& rp = reports[0];
    std::memset(&rp, 0, sizeof rp);
    rp.level = 1;
    rp.r = r;
    rp.max_load = *std::max_element(m->new_sizes.begin(), m->new_sizes.end());
    rp.min_load = *std::min_element(m->new_sizes.begin(), m->new_sizes.end());
    rp.sample_size = S;
    rp.plan_load = m->max_load;
    rp.over_budget = m->max_load > (uint64_t)std::ceil((1.0 + eps_l) * (double)n / r);
    rp.max_words = m->stats[0]; rp.max_msgs = m->stats[1];
    rp.max_sent_msgs = m->stats[2]; rp.max_recv_msgs = m->stats[3];
  }
  // ---- later levels and final sort: one continuation per device ---------
  std::vector<std::vector<ams_level_report_t>> reps(G, std::vector<ams_level_report_t>(k));
  rc = for_devices(G, [&](int i) -> int {
    ams_params_t q = *prm;
    q.oversampling = a;
    q.level_base = 1;
    q.init_groups = gpr;
    q.pe_base = i * pl;
    return ams_sort_run(m->ctx[i], &q, pl, m->new_sizes.data() + (size_t)i * pl, src_k[i], src_v[i], out[i],
                        out_vals ? out_vals[i] : nullptr, out_pe_sizes ? out_pe_sizes + (size_t)i * pl : nullptr,
                        reps[i].data());
  });
  if (rc) return rc;
  if (reports) {
    for (int lv = 1; lv < k; ++lv) {
      ams_level_report_t& rp = reports[lv];
      rp = reps[0][lv];
      for (int i = 1; i < G; ++i) {
        const ams_level_report_t& o = reps[i][lv];
        rp.max_load = std::max(rp.max_load, o.max_load);
        rp.min_load = std::min(rp.min_load, o.min_load);
        rp.sample_size = std::max(rp.sample_size, o.sample_size);
        rp.plan_load = std::max(rp.plan_load, o.plan_load);
        rp.over_budget += o.over_budget;
        rp.max_words = std::max(rp.max_words, o.max_words);
        rp.max_msgs = std::max(rp.max_msgs, o.max_msgs);
        rp.max_sent_msgs = std::max(rp.max_sent_msgs, o.max_sent_msgs);
        rp.max_recv_msgs = std::max(rp.max_recv_msgs, o.max_recv_msgs);
      }
    }
  }
  return sync_all(m);
}

int ams_mg_level1_dims(const ams_mg_t* m, int* r, int* p, int* nb_stride) {
  if (!m) return set_error(AMS_EINVAL, "null argument");
  if (r) *r = m->r;
  if (p) *p = m->p;
  if (nb_stride) *nb_stride = m->nb_stride;
  return AMS_OK;
}

int ams_mg_level1(const ams_mg_t* m, uint64_t* sizes_before, uint64_t* drawn, int32_t* nb, uint32_t* seg_hist,
                  uint64_t* boundaries, uint64_t* loads, uint64_t* max_load, uint64_t* new_sizes,
                  uint64_t* stats) {
  if (!m) return set_error(AMS_EINVAL, "null argument");
  auto put = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
  };
  put(sizes_before, m->sizes_before);
  if (drawn) *drawn = m->drawn;
  if (nb) *nb = m->nb;
  put(seg_hist, m->hist);
  put(boundaries, m->boundaries);
  put(loads, m->loads);
  if (max_load) *max_load = m->max_load;
  put(new_sizes, m->new_sizes);
  put(stats, m->stats);
  return AMS_OK;
}

}  // extern "C"
