// Consecutive-bucket grouping and the per-level delivery bookkeeping,
// restated natively.
//
// Reference: _scan / scan_groups / optimal_group_plan (ams.py:78-154), the
// simple delivery's quota slots (delivery.py:78-106, 138-180), the
// deterministic delivery's member assignment (delivery.py:188-306) and the
// exchange shape Network.exchange records (simnet.py:294-335).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../ams_host.h"

namespace ams {
namespace {

struct Plan {
  std::vector<uint64_t> boundaries, loads;
  uint64_t max_load = 0;
};

// _scan (ams.py:78-109): returns feasibility; `overflow` = smallest
// load+bucket that failed to fit (UINT64_MAX when none).
bool scan(const uint64_t* sizes, int nb, int r, uint64_t limit, Plan* plan, uint64_t* overflow) {
  uint64_t ovf = UINT64_MAX;
  plan->boundaries.assign(1, 0);
  plan->loads.clear();
  uint64_t cur = 0;
  for (int i = 0; i < nb; ++i) {
    const uint64_t size = sizes[i];
    if (size > limit) { *overflow = ovf; return false; }
    if (cur + size > limit) {
      if (cur + size < ovf) ovf = cur + size;
      plan->boundaries.push_back((uint64_t)i);
      plan->loads.push_back(cur);
      cur = size;
    } else {
      cur += size;
    }
  }
  plan->boundaries.push_back((uint64_t)nb);
  plan->loads.push_back(cur);
  *overflow = ovf;
  if ((int)plan->loads.size() > r) return false;
  while ((int)plan->loads.size() < r) {
    plan->boundaries.push_back((uint64_t)nb);
    plan->loads.push_back(0);
  }
  plan->max_load = *std::max_element(plan->loads.begin(), plan->loads.end());
  return true;
}

// optimal_group_plan (ams.py:119-154), including the float window bound.
void optimal_plan(const uint64_t* sizes, int nb, int r, Plan* best) {
  uint64_t total = 0, mx = 0;
  for (int i = 0; i < nb; ++i) { total += sizes[i]; mx = std::max(mx, sizes[i]); }
  uint64_t lo = std::max(mx, (total + r - 1) / (uint64_t)r);
  const int b_est = std::max(1, nb / r);
  const double est = (double)total / (double)r * (1.0 + 4.0 / (double)b_est);
  uint64_t hi = std::max(lo, (uint64_t)std::ceil(est));
  Plan plan;
  uint64_t overflow;
  bool ok = scan(sizes, nb, r, hi, &plan, &overflow);
  if (!ok) {
    lo = std::max(lo, overflow != UINT64_MAX ? overflow : hi + 1);
    hi = total;
    scan(sizes, nb, r, hi, &plan, &overflow);  // one group of everything fits
  }
  hi = plan.max_load;
  *best = plan;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    ok = scan(sizes, nb, r, mid, &plan, &overflow);
    if (ok) {
      hi = plan.max_load;
      *best = plan;
    } else {
      lo = overflow != UINT64_MAX ? overflow : mid + 1;
    }
  }
}

// Exchange shape of deliver_simple for one group (see oracle
// _exchange_stats): pieces[j][g], P members, r subgroups of P/r.
void exchange_stats(const std::vector<uint64_t>& pieces, int P, int r, uint64_t out[4]) {
  const int sub = P / r;
  std::vector<uint64_t> sw(P, 0), rw(P, 0), sm(P, 0), rm(P, 0);
  for (int g = 0; g < r; ++g) {
    uint64_t m = 0;
    for (int j = 0; j < P; ++j) m += pieces[(size_t)j * r + g];
    uint64_t start = 0;
    for (int j = 0; j < P; ++j) {
      const uint64_t size = pieces[(size_t)j * r + g];
      if (size == 0 || m == 0) { start += size; continue; }
      // First owner of element number `start` (delivery.py:94).
      int t = (int)(((unsigned __int128)(start + 1) * sub + m - 1) / m) - 1;
      uint64_t covered = 0;
      while (covered < size && t < sub) {
        const uint64_t slot_hi = (uint64_t)(((unsigned __int128)m * (t + 1)) / sub);
        const int64_t take = (int64_t)std::min(start + size, slot_hi) - (int64_t)(start + covered);
        if (take > 0) {
          const int dest = g * sub + t;
          if (dest != j) { sw[j] += take; rw[dest] += take; sm[j] += 1; rm[dest] += 1; }
          covered += (uint64_t)take;
        }
        ++t;
      }
      start += size;
    }
  }
  uint64_t hs = 0, hr = 0, ms = 0, mr = 0;
  for (int j = 0; j < P; ++j) {
    hs = std::max(hs, sw[j]); hr = std::max(hr, rw[j]);
    ms = std::max(ms, sm[j]); mr = std::max(mr, rm[j]);
  }
  out[0] = std::max(hs, hr);
  out[1] = std::max(ms, mr);
  out[2] = ms;
  out[3] = mr;
}

// feistel_new(n, SeedSpec(master, stream)).apply(i) for every i
// (core.py:96-159): four rounds (lo, hi) -> (hi, (lo + T_k[hi]) mod side)
// over side^2 >= n, T_k[v] = splitmix64(v ^ key64(k)) mod side, cycle
// walking values >= n; key64(k) = first 8 bytes (big endian) of
// blake2b-128("{master}\x1f{stream}\x1fk{k}") (core.py:69-71).
std::vector<uint64_t> feistel_perm(uint64_t n, int64_t master_seed, const std::string& stream) {
  uint64_t side = (uint64_t)std::sqrt((double)n);
  while (side * side > n) --side;
  while (side * side < n) ++side;
  auto mix64 = [](uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
  };
  std::vector<uint64_t> tables(4 * side), perm(n);
  for (int i = 0; i < 4; ++i) {
    const std::string text = std::to_string(master_seed) + "\x1f" + stream + "\x1fk" + std::to_string(i);
    uint8_t d[16];
    blake2b_128(reinterpret_cast<const uint8_t*>(text.data()), text.size(), d);
    uint64_t key = 0;
    for (int b = 0; b < 8; ++b) key = (key << 8) | d[b];
    for (uint64_t v = 0; v < side; ++v) tables[i * side + v] = mix64(v ^ key) % side;
  }
  for (uint64_t j = 0; j < n; ++j) {
    uint64_t x = j;
    for (uint64_t it = 0; it < side * side; ++it) {
      uint64_t hi = x / side, lo = x % side;
      for (int i = 0; i < 4; ++i) {
        const uint64_t nhi = (lo + tables[i * side + hi]) % side;
        lo = hi;
        hi = nhi;
      }
      x = lo + hi * side;
      if (x < n) break;
    }
    perm[j] = x;
  }
  return perm;
}

// sorted(range(n), key=feistel.apply): the enumeration order (delivery.py:131-134).
std::vector<int> feistel_order(int n, int64_t master_seed, const std::string& stream) {
  const std::vector<uint64_t> perm = feistel_perm((uint64_t)n, master_seed, stream);
  std::vector<int> order(n);
  for (int j = 0; j < n; ++j) order[j] = j;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return perm[a] < perm[b]; });
  return order;
}

// _slice_range (delivery.py:83-106): numbers [start, start + size) of a
// subgroup with m numbers over `sub` members -> cuts (piece offset base + ...).
bool slice_range(int j, int g, int sub, uint64_t m, uint64_t start, uint64_t size, uint64_t base,
                 std::vector<struct Cut>& cuts);

// One slice of a delivery: elements [off, off + len) of piece (member j,
// subgroup g) go to member t of subgroup g.
struct Cut { int j, g, t; uint64_t off, len; };

// Slices -> {src, dst, len} (src in the group's simple layout: subgroup,
// source member, bucket; dst in the new member arrays, receivers
// concatenating by source, simnet.py:324-325), new member sizes and the
// data-exchange shape (simnet.py:294-335).
bool slice_range(int j, int g, int sub, uint64_t m, uint64_t start, uint64_t size, uint64_t base,
                 std::vector<Cut>& cuts) {
  if (size == 0 || m == 0) return true;
  int t = (int)((((unsigned __int128)(start + 1) * sub + m - 1) / m) - 1);
  uint64_t covered = 0;
  while (covered < size && t < sub) {
    const uint64_t hi = (uint64_t)(((unsigned __int128)m * (t + 1)) / sub);
    const int64_t take = (int64_t)std::min(start + size, hi) - (int64_t)(start + covered);
    if (take > 0) {
      cuts.push_back({j, g, t, base + covered, (uint64_t)take});
      covered += (uint64_t)take;
    }
    ++t;
  }
  return covered == size;
}

int emit_slices(int P, int r, const uint64_t* pieces, const std::vector<Cut>& cuts,
                uint64_t* out_new_sizes, uint64_t* out_slices, int slice_cap, int* out_nslices,
                uint64_t* out_stats) {
  const int sub = P / r;
  if ((int)cuts.size() > slice_cap) return set_error(AMS_EINTERNAL, "slice buffer too small");
  // New member sizes and receive order (by source member).
  std::vector<uint64_t> ns(P, 0);
  for (const Cut& c : cuts) ns[(size_t)c.g * sub + c.t] += c.len;
  std::vector<uint64_t> mbase(P + 1, 0);
  for (int d = 0; d < P; ++d) mbase[d + 1] = mbase[d] + ns[d];
  std::vector<uint64_t> gstart(r + 1, 0), pstart((size_t)P * r, 0);
  for (int g = 0; g < r; ++g) {
    uint64_t run = gstart[g];
    for (int j = 0; j < P; ++j) { pstart[(size_t)j * r + g] = run; run += pieces[(size_t)j * r + g]; }
    gstart[g + 1] = run;
  }
  std::vector<int> order(cuts.size());
  for (size_t i = 0; i < cuts.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    const int da = cuts[a].g * sub + cuts[a].t, db = cuts[b].g * sub + cuts[b].t;
    if (da != db) return da < db;
    return cuts[a].j != cuts[b].j ? cuts[a].j < cuts[b].j : cuts[a].off < cuts[b].off;
  });
  std::vector<uint64_t> fill(P, 0);
  std::vector<uint64_t> sw(P, 0), rw(P, 0), sm(P, 0), rm(P, 0);
  int k = 0;
  for (int i : order) {
    const Cut& c = cuts[i];
    const int d = c.g * sub + c.t;
    out_slices[3 * k + 0] = pstart[(size_t)c.j * r + c.g] + c.off;
    out_slices[3 * k + 1] = mbase[d] + fill[d];
    out_slices[3 * k + 2] = c.len;
    fill[d] += c.len;
    if (c.len > 0 && d != c.j) { sw[c.j] += c.len; rw[d] += c.len; sm[c.j] += 1; rm[d] += 1; }
    ++k;
  }
  *out_nslices = k;
  std::copy(ns.begin(), ns.end(), out_new_sizes);
  if (out_stats) {
    uint64_t hs = 0, hr = 0, ms = 0, mr = 0;
    for (int j = 0; j < P; ++j) {
      hs = std::max(hs, sw[j]); hr = std::max(hr, rw[j]);
      ms = std::max(ms, sm[j]); mr = std::max(mr, rm[j]);
    }
    out_stats[0] = std::max(hs, hr);
    out_stats[1] = std::max(ms, mr);
    out_stats[2] = ms;
    out_stats[3] = mr;
  }
  return AMS_OK;
}

}  // namespace
}  // namespace ams

using namespace ams;

extern "C" {

int ams_scan_groups(const uint64_t* sizes, int nb, int r, uint64_t limit,
                    uint64_t* out_boundaries, uint64_t* out_loads, uint64_t* out_max_load) {
  if (nb < 1 || r < 1) return set_error(AMS_EINVAL, "bad histogram / group count");
  Plan plan;
  uint64_t ovf;
  if (!scan(sizes, nb, r, limit, &plan, &ovf)) return 1;  // infeasible (not an error)
  std::copy(plan.boundaries.begin(), plan.boundaries.end(), out_boundaries);
  std::copy(plan.loads.begin(), plan.loads.end(), out_loads);
  *out_max_load = plan.max_load;
  return AMS_OK;
}

int ams_group_plan(const uint64_t* sizes, int nb, int r, uint64_t* out_boundaries,
                   uint64_t* out_loads, uint64_t* out_max_load) {
  if (r < 1) return set_error(AMS_EINVAL, "need at least one group");
  if (nb < 1) return set_error(AMS_EINVAL, "histogram has no buckets");
  Plan plan;
  optimal_plan(sizes, nb, r, &plan);
  std::copy(plan.boundaries.begin(), plan.boundaries.end(), out_boundaries);
  std::copy(plan.loads.begin(), plan.loads.end(), out_loads);
  *out_max_load = plan.max_load;
  return AMS_OK;
}

// The host half of one level (ams.py:231-256) for every group, given the
// per-member bucket histograms.
//   seg_hist: [sum(group_npe)][nb_stride] u32, members group-major.
//   Per group g (npe P, nb buckets, r groups): boundaries (r+1), loads (r),
//   max_load; per member the next-level size (quota slots of the subgroup,
//   delivery.py:78-80); 4 exchange stats (max_words, max_msgs,
//   max_sent_msgs, max_recv_msgs).
int ams_plan_level(int ngroups, const int32_t* group_npe, const int32_t* group_nb, int r,
                   const uint32_t* seg_hist, int nb_stride, uint64_t* out_boundaries,
                   uint64_t* out_loads, uint64_t* out_max_load, uint64_t* out_new_sizes,
                   uint64_t* out_stats) {
  if (r < 1) return set_error(AMS_EINVAL, "need at least one group");
  size_t seg0 = 0;
  std::vector<uint64_t> h, pieces;
  for (int g = 0; g < ngroups; ++g) {
    const int P = group_npe[g], nb = group_nb[g];
    if (P % r != 0) {
      return set_error(AMS_EINVAL, std::to_string(P) + " PEs cannot form " +
                                       std::to_string(r) + " groups");
    }
    if (nb < 1 || nb > nb_stride) return set_error(AMS_EINVAL, "bad bucket count");
    h.assign(nb, 0);
    for (int j = 0; j < P; ++j)
      for (int b = 0; b < nb; ++b) h[b] += seg_hist[(seg0 + j) * nb_stride + b];
    Plan plan;
    optimal_plan(h.data(), nb, r, &plan);
    std::copy(plan.boundaries.begin(), plan.boundaries.end(), out_boundaries + (size_t)g * (r + 1));
    std::copy(plan.loads.begin(), plan.loads.end(), out_loads + (size_t)g * r);
    out_max_load[g] = plan.max_load;
    const int sub = P / r;
    for (int gg = 0; gg < r; ++gg) {
      const uint64_t m = plan.loads[gg];
      for (int t = 0; t < sub; ++t) {
        const uint64_t a = (uint64_t)(((unsigned __int128)m * t) / sub);
        const uint64_t b = (uint64_t)(((unsigned __int128)m * (t + 1)) / sub);
        out_new_sizes[seg0 + (size_t)gg * sub + t] = b - a;
      }
    }
    if (out_stats) {
      pieces.assign((size_t)P * r, 0);
      for (int j = 0; j < P; ++j)
        for (int gg = 0; gg < r; ++gg) {
          uint64_t s = 0;
          for (uint64_t b = plan.boundaries[gg]; b < plan.boundaries[gg + 1]; ++b)
            s += seg_hist[(seg0 + j) * nb_stride + b];
          pieces[(size_t)j * r + gg] = s;
        }
      exchange_stats(pieces, P, r, out_stats + (size_t)g * 4);
    }
    seg0 += P;
  }
  return AMS_OK;
}

// deliver_simple (delivery.py:151-180) for one group from its piece sizes
// [P][r]: the member arrays are consecutive slices of the group's simple
// layout (no relayout), so only the new member sizes (quota slots,
// delivery.py:78-80) and the exchange stats are produced.
int ams_deliver_simple(int P, int r, const uint64_t* pieces, uint64_t* out_new_sizes,
                       uint64_t* out_stats) {
  if (r < 1 || P < 1 || P % r != 0)
    return set_error(AMS_EINVAL, std::to_string(P) + " PEs cannot form " + std::to_string(r) + " groups");
  if (!pieces || !out_new_sizes) return set_error(AMS_EINVAL, "null argument");
  const int sub = P / r;
  for (int g = 0; g < r; ++g) {
    uint64_t m = 0;
    for (int j = 0; j < P; ++j) m += pieces[(size_t)j * r + g];
    for (int t = 0; t < sub; ++t) {
      const uint64_t a = (uint64_t)(((unsigned __int128)m * t) / sub);
      const uint64_t b = (uint64_t)(((unsigned __int128)m * (t + 1)) / sub);
      out_new_sizes[(size_t)g * sub + t] = b - a;
    }
  }
  if (out_stats) exchange_stats(std::vector<uint64_t>(pieces, pieces + (size_t)P * r), P, r, out_stats);
  return AMS_OK;
}

// deliver_deterministic (delivery.py:188-306) for one group of P members
// and r subgroups (members [g*P/r, (g+1)*P/r) form subgroup g), from the
// piece sizes [P][r] (member j's buckets of group g).  Small pieces
// (size*2*P*r <= n) go whole to member small_index / r of their subgroup;
// large pieces fill the members' residual quota capacities in member order
// (the merge of two prefix sums), so one piece spans consecutive members.
// Receivers concatenate in source order (simnet.py:324-325).  Output, per
// slice: {src, dst, len} with src relative to the start of the group's
// simple layout (subgroup-major, then source member, then bucket) and dst
// relative to the start of the group's new member arrays; new_sizes [P];
// stats [4] as ams_plan_level (NULL: skip).
int ams_deliver_deterministic(int P, int r, int pe0, const uint64_t* pieces, uint64_t* out_new_sizes,
                              uint64_t* out_slices, int slice_cap, int* out_nslices,
                              uint64_t* out_stats) {
  if (P < 1 || r < 1 || P % r != 0)
    return set_error(AMS_EINVAL, std::to_string(P) + " PEs cannot form " + std::to_string(r) + " groups");
  const int sub = P / r;
  unsigned __int128 n = 0;
  for (int i = 0; i < P * r; ++i) n += pieces[i];
  const uint64_t cap = (uint64_t)((n + (unsigned)P - 1) / (unsigned)P);  // ceil(n/p)
  for (int j = 0; j < P; ++j)
    for (int g = 0; g < r; ++g)
      if (pieces[(size_t)j * r + g] > cap)
        return set_error(AMS_EINVAL, "piece (" + std::to_string(pe0 + j) + "," + std::to_string(g) +
                                         ") larger than ceil(n/p): " +
                                         std::to_string(pieces[(size_t)j * r + g]) + " > " +
                                         std::to_string(cap));
  auto is_small = [&](uint64_t size) {
    return (unsigned __int128)size * 2u * (unsigned)P * (unsigned)r <= n;
  };
  std::vector<Cut> cuts;
  for (int g = 0; g < r; ++g) {
    uint64_t m_g = 0;
    for (int j = 0; j < P; ++j) m_g += pieces[(size_t)j * r + g];
    std::vector<int64_t> small_load(sub, 0);
    std::vector<std::pair<int, uint64_t>> larges;
    uint64_t small_index = 0;
    for (int j = 0; j < P; ++j) {
      const uint64_t size = pieces[(size_t)j * r + g];
      if (size == 0) continue;
      if (!is_small(size)) { larges.push_back({j, size}); continue; }
      const int t = (int)(small_index / (uint64_t)r);
      ++small_index;
      small_load[t] += (int64_t)size;
      cuts.push_back({j, g, t, 0, size});
    }
    std::vector<uint64_t> bounds(sub + 1, 0);
    for (int t = 0; t < sub; ++t) {
      const uint64_t lo = (uint64_t)(((unsigned __int128)m_g * t) / sub);
      const uint64_t hi = (uint64_t)(((unsigned __int128)m_g * (t + 1)) / sub);
      const int64_t res = std::max<int64_t>(0, (int64_t)(hi - lo) - small_load[t]);
      bounds[t + 1] = bounds[t] + (uint64_t)res;
    }
    uint64_t pos = 0;
    for (const auto& [j, size] : larges) {
      // bisect_right(bounds, pos) - 1
      int t = (int)(std::upper_bound(bounds.begin(), bounds.end(), pos) - bounds.begin()) - 1;
      uint64_t covered = 0;
      while (covered < size) {
        if (t >= sub) return set_error(AMS_EINTERNAL, "residual capacities cannot hold the large pieces");
        const int64_t take = (int64_t)std::min(pos + size, bounds[t + 1]) - (int64_t)(pos + covered);
        if (take > 0) {
          cuts.push_back({j, g, t, covered, (uint64_t)take});
          covered += (uint64_t)take;
        }
        ++t;
      }
      pos += size;
    }
  }
  return emit_slices(P, r, pieces, cuts, out_new_sizes, out_slices, slice_cap, out_nslices, out_stats);
}

// deliver_simple_permuted (delivery.py:151-185): subgroup g enumerates the
// sending members in the order sorted(range(P), key=feistel.apply) of the
// seeded permutation of stream "{level_stream}/deliver/order-g{g}"
// (core.py:96-159: four keyed digit-pair rounds over side^2, cycle
// walking); member t owns numbers [m t / p', m (t+1) / p') of it.  Output
// as ams_deliver_deterministic.
int ams_deliver_permuted(int P, int r, int64_t master_seed, const char* level_stream,
                         const uint64_t* pieces, uint64_t* out_new_sizes, uint64_t* out_slices,
                         int slice_cap, int* out_nslices, uint64_t* out_stats) {
  if (P < 1 || r < 1 || P % r != 0)
    return set_error(AMS_EINVAL, std::to_string(P) + " PEs cannot form " + std::to_string(r) + " groups");
  if (!level_stream) return set_error(AMS_EINVAL, "null stream id");
  const int sub = P / r;
  std::vector<Cut> cuts;
  for (int g = 0; g < r; ++g) {
    const std::vector<int> order =
        feistel_order(P, master_seed, std::string(level_stream) + "/deliver/order-g" + std::to_string(g));
    uint64_t m = 0;
    for (int j = 0; j < P; ++j) m += pieces[(size_t)j * r + g];
    uint64_t start = 0;
    for (int j : order) {
      const uint64_t size = pieces[(size_t)j * r + g];
      if (!slice_range(j, g, sub, m, start, size, 0, cuts))
        return set_error(AMS_EINTERNAL, "quota mapping failed to cover a piece");
      start += size;
    }
  }
  return emit_slices(P, r, pieces, cuts, out_new_sizes, out_slices, slice_cap, out_nslices, out_stats);
}

// deliver_randomized (delivery.py:318-436) with the default delegation
// factor (309-315): pieces above s = ceil(a n / (r p)) are cut into
// s-element chunks plus a remainder; full chunks go to holder
// feistel(rank) % p ("…/deliver/delegate"); subgroup g numbers its chunks
// holder by holder in the Feistel order of "…/deliver/order-g{g}", each
// holder's chunks in Random("…/deliver/reorder-g{g}-h{holder}").shuffle
// order (CPython's shuffle over MT19937 randbelow); members own quota
// slots of that numbering.  Output as ams_deliver_deterministic.
int ams_deliver_randomized(int P, int r, int64_t master_seed, const char* level_stream,
                           const uint64_t* pieces, uint64_t* out_new_sizes, uint64_t* out_slices,
                           int slice_cap, int* out_nslices, uint64_t* out_stats) {
  if (P < 1 || r < 1 || P % r != 0)
    return set_error(AMS_EINVAL, std::to_string(P) + " PEs cannot form " + std::to_string(r) + " groups");
  if (!level_stream) return set_error(AMS_EINVAL, "null stream id");
  const int sub = P / r;
  uint64_t n = 0;
  for (int i = 0; i < P * r; ++i) n += pieces[i];
  uint64_t a = 1;
  if ((uint64_t)r * P > 2) {
    const double x = 0.5 * (std::sqrt(1.0 + r / std::log(r * (double)P / 2.0)) - 1.0);
    a = std::max<uint64_t>(1, (uint64_t)std::floor(x));
  }
  const uint64_t rp = (uint64_t)r * P;
  const uint64_t s = std::max<uint64_t>(1, (a * n + rp - 1) / rp);
  struct Chunk { int j, g; uint64_t off, len; bool large; };
  std::vector<Chunk> chunks;
  for (int j = 0; j < P; ++j)
    for (int g = 0; g < r; ++g) {
      const uint64_t size = pieces[(size_t)j * r + g];
      if (size == 0) continue;
      if (size > s) {
        const uint64_t whole = size / s, rem = size % s;
        for (uint64_t c = 0; c < whole; ++c) chunks.push_back({j, g, c * s, s, true});
        if (rem) chunks.push_back({j, g, whole * s, rem, false});
      } else {
        chunks.push_back({j, g, 0, size, false});
      }
    }
  const std::string ds = std::string(level_stream) + "/deliver";
  std::vector<int> holder(chunks.size());
  for (size_t i = 0; i < chunks.size(); ++i) holder[i] = chunks[i].j;
  std::vector<size_t> large;
  for (size_t i = 0; i < chunks.size(); ++i)
    if (chunks[i].large) large.push_back(i);
  if (!large.empty()) {
    const std::vector<uint64_t> perm = feistel_perm(large.size(), master_seed, ds + "/delegate");
    for (size_t rank = 0; rank < large.size(); ++rank) holder[large[rank]] = (int)(perm[rank] % (uint64_t)P);
  }
  std::vector<std::vector<size_t>> held((size_t)r * P);
  for (size_t i = 0; i < chunks.size(); ++i) held[(size_t)chunks[i].g * P + holder[i]].push_back(i);
  std::vector<uint64_t> start_of(chunks.size(), 0), totals(r, 0);
  for (int g = 0; g < r; ++g) {
    uint64_t running = 0;
    for (int h : feistel_order(P, master_seed, ds + "/order-g" + std::to_string(g))) {
      std::vector<size_t>& mine = held[(size_t)g * P + h];
      if (mine.empty()) continue;
      uint32_t words[4];
      const int nw = stream_seed_words(std::to_string(master_seed) + "\x1f" + ds + "/reorder-g" +
                                           std::to_string(g) + "-h" + std::to_string(h) + "\x1f",
                                       words);
      Mt19937 rng;
      rng.init_by_array(words, nw);
      for (size_t i = mine.size() - 1; i >= 1; --i) {  // Random.shuffle
        const size_t k = (size_t)rng.randbelow(i + 1);
        std::swap(mine[i], mine[k]);
      }
      for (size_t cid : mine) {
        start_of[cid] = running;
        running += chunks[cid].len;
      }
    }
    totals[g] = running;
  }
  std::vector<Cut> cuts;
  for (size_t cid = 0; cid < chunks.size(); ++cid) {
    const Chunk& ch = chunks[cid];
    if (!slice_range(ch.j, ch.g, sub, totals[ch.g], start_of[cid], ch.len, ch.off, cuts))
      return set_error(AMS_EINTERNAL, "quota mapping failed to cover a piece");
  }
  return emit_slices(P, r, pieces, cuts, out_new_sizes, out_slices, slice_cap, out_nslices, out_stats);
}

}  // extern "C"
