// mg_adapt.cpp — refine / coarsen / 2:1 balance of the block forest (
// PAPER.md §2.1; reading A2).  Host code on the leaf list (a
// few 10^4 blocks): the data-parallel part of adaptation is the detail kernel
// (mg_adapt.cu).
//
//  (1) refine every leaf with γ > ε_r below max_level ("A grid block is refined into 8
//      finer blocks whenever … γ above ε_r"); leaves touching an unbounded face stay
//      at level 0 unless U1 is allowed — such refinements are suppressed and
//      counted;
//  (2) coarsen every complete octet of leaves, none refined in (1), all γ < ε_c ("when
//      all 8 blocks involve detail coefficients below … ε_c, they revert back to a
//      single grid block"), whose parent keeps the 2:1 constraint with the grid of (1);
//  (3) balance by refinement ("two adjacent blocks cannot have a resolution jump larger
//      than one level"): until, for every leaf of level m >= 2, the parent of each of
//      its 26 neighbours exists as a block, refine the leaf covering a missing one;
//      if that leaf may not be refined (unbounded face), the parent of the leaf that
//      needs it is barred from refinement and the pass restarts from the input.
#include <algorithm>
#include <array>
#include <cstdint>
#include <map>
#include <set>
#include <vector>

#include "mg.h"

namespace {

using Key = std::array<int32_t, 4>;  // level, x, y, z

struct Forest {
  int nb0[3];
  bool per[3];
  bool allow;
  int64_t nb(int lev, int a) const { return (int64_t)nb0[a] << lev; }
  bool wrap(int lev, int64_t c[3]) const {
    for (int a = 0; a < 3; ++a) {
      const int64_t n = nb(lev, a);
      if (per[a]) c[a] = ((c[a] % n) + n) % n;
      else if (c[a] < 0 || c[a] >= n) return false;
    }
    return true;
  }
  bool touches_unbounded(const Key& k) const {
    for (int a = 0; a < 3; ++a)
      if (!per[a] && (k[1 + a] == 0 || k[1 + a] == nb(k[0], a) - 1)) return true;
    return false;
  }
};

void children(const Key& k, Key out[8]) {
  int n = 0;
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) out[n++] = {k[0] + 1, 2 * k[1] + dx, 2 * k[2] + dy, 2 * k[3] + dz};
}

Key parent(const Key& k) { return {k[0] - 1, k[1] >> 1, k[2] >> 1, k[3] >> 1}; }

void add_with_ancestors(std::set<Key>& blocks, Key k) {
  while (k[0] >= 0) {
    if (!blocks.insert(k).second) break;  // ancestors already present
    if (k[0] == 0) break;
    k = parent(k);
  }
}

// One pass of steps (1)-(3) with the blocks in `forbidden` barred from refinement.
// Returns true and fills `out`, or false and sets `bad` = the parent of the leaf whose
// 2:1 neighbourhood would need a frozen block refined.
bool adapt_once(const Forest& F, const std::set<Key>& L, const std::map<Key, double>& gam, double eps_r,
                double eps_c, int max_level, const std::set<Key>& forbidden, std::set<Key>& out, Key& bad,
                int32_t& suppressed) {
  auto frozen = [&](const Key& k) { return (F.touches_unbounded(k) && !F.allow) || forbidden.count(k) > 0; };
  suppressed = 0;
  // (1) refinement
  std::set<Key> refine;
  for (const Key& k : L) {
    if (!(gam.at(k) > eps_r) || k[0] >= max_level) continue;
    if (frozen(k)) {
      ++suppressed;
      continue;
    }
    refine.insert(k);
  }
  std::set<Key> L1;
  for (const Key& k : L)
    if (!refine.count(k)) L1.insert(k);
  for (const Key& k : refine) {
    Key ch[8];
    children(k, ch);
    for (auto& c : ch) L1.insert(c);
  }
  std::set<Key> blocks1;
  for (const Key& k : L1) add_with_ancestors(blocks1, k);
  // (2) coarsening of complete octets
  std::map<Key, std::vector<Key>> parents;
  for (const Key& k : L)
    if (k[0] > 0 && !refine.count(k)) parents[parent(k)].push_back(k);
  std::vector<Key> coarsen;
  for (const auto& pk : parents) {
    const Key& p = pk.first;
    const auto& kids = pk.second;
    if (kids.size() != 8) continue;
    bool ok = true;
    for (const Key& c : kids) ok = ok && gam.at(c) < eps_c;
    if (!ok) continue;
    for (int o = 0; o < 27 && ok; ++o) {
      if (o == 13) continue;
      int64_t q[3] = {(int64_t)p[1] + o % 3 - 1, (int64_t)p[2] + (o / 3) % 3 - 1, (int64_t)p[3] + o / 9 - 1};
      if (!F.wrap(p[0], q)) continue;
      const Key qk = {p[0], (int32_t)q[0], (int32_t)q[1], (int32_t)q[2]};
      Key ch[8];
      children(qk, ch);
      for (auto& c : ch)  // blocks two levels finer than p next to p
        if (blocks1.count(Key{c[0] + 1, 2 * c[1], 2 * c[2], 2 * c[3]})) ok = false;
    }
    if (ok) coarsen.push_back(p);
  }
  std::set<Key> L2 = L1;
  for (const Key& p : coarsen) {
    Key ch[8];
    children(p, ch);
    for (auto& c : ch) L2.erase(c);
    L2.insert(p);
  }
  // (3) 2:1 balance by refinement
  std::set<Key> blocks;
  for (const Key& k : L2) add_with_ancestors(blocks, k);
  bool changed = true;
  while (changed) {
    changed = false;
    const std::vector<Key> snap(L2.begin(), L2.end());
    for (const Key& lf : snap) {
      if (!L2.count(lf) || lf[0] < 2) continue;
      const int m = lf[0] - 1;
      for (int o = 0; o < 27; ++o) {
        if (o == 13) continue;
        int64_t n[3] = {(int64_t)lf[1] + o % 3 - 1, (int64_t)lf[2] + (o / 3) % 3 - 1, (int64_t)lf[3] + o / 9 - 1};
        if (!F.wrap(lf[0], n)) continue;
        // the region of neighbour n must be covered by blocks of level >= m
        const Key qk = {m, (int32_t)(n[0] >> 1), (int32_t)(n[1] >> 1), (int32_t)(n[2] >> 1)};
        if (blocks.count(qk)) continue;
        Key a = qk;
        while (a[0] > 0 && !L2.count(a)) a = parent(a);
        if (!L2.count(a)) return false;  // not covered: rejected by validate() beforehand
        if (frozen(a)) {
          bad = parent(lf);
          return false;
        }
        L2.erase(a);
        Key ch[8];
        children(a, ch);
        for (auto& c : ch) {
          L2.insert(c);
          blocks.insert(c);
        }
        changed = true;
      }
    }
  }
  out.swap(L2);
  return true;
}

// Input checks: no duplicate leaf, no leaf with a descendant, complete
// octets, level 0 covered, no refined leaf on an unbounded face unless U1.  An input
// that is not 2:1 balanced is accepted (step (3) balances it).  MG_OK or the MG_ERR_*
// code of the first violation.
int validate(const Forest& F, const std::set<Key>& L, int64_t n_in) {
  if ((int64_t)L.size() != n_in) return MG_ERR_LAYOUT_NESTING;  // duplicates
  std::set<Key> blocks;
  for (const Key& k : L) {
    if (k[0] < 0 || k[0] > 20) return MG_ERR_ARG;
    for (int a = 0; a < 3; ++a)
      if (k[1 + a] < 0 || k[1 + a] >= F.nb(k[0], a)) return MG_ERR_ARG;
    add_with_ancestors(blocks, k);
  }
  for (const Key& k : L) {
    Key ch[8];
    children(k, ch);
    for (auto& c : ch)
      if (blocks.count(c)) return MG_ERR_LAYOUT_NESTING;  // a leaf that is also refined
  }
  for (const Key& b : blocks) {
    if (L.count(b)) continue;
    Key ch[8];
    children(b, ch);
    for (auto& c : ch)
      if (!blocks.count(c)) return MG_ERR_LAYOUT_NESTING;  // partially refined block
  }
  int64_t n0 = 0;
  for (const Key& b : blocks) n0 += b[0] == 0;
  if (n0 != (int64_t)F.nb0[0] * F.nb0[1] * F.nb0[2]) return MG_ERR_LAYOUT_NESTING;
  for (const Key& k : L) {
    if (k[0] > 0 && !F.allow && F.touches_unbounded(k)) return MG_ERR_UNBOUNDED_REFINED;
  }
  return MG_OK;
}

}  // namespace

extern "C" int mg_adapt(const int32_t base_blocks[3], const int32_t bc[6], int32_t allow_unbounded_refined,
                        const int32_t* leaves, int32_t n_leaf, const double* gamma, double eps_r, double eps_c,
                        int32_t max_level, int32_t* out_leaves, int32_t out_capacity, int32_t* n_out,
                        int32_t* n_suppressed) {
  if (!base_blocks || !bc || n_leaf < 0 || (n_leaf > 0 && (!leaves || !gamma)) || !n_out || max_level < 0)
    return MG_ERR_ARG;
  Forest F;
  for (int a = 0; a < 3; ++a) {
    if (base_blocks[a] <= 0) return MG_ERR_ARG;
    F.nb0[a] = base_blocks[a];
    F.per[a] = bc[2 * a] == MG_BC_PERIODIC;
  }
  F.allow = allow_unbounded_refined != 0;
  std::set<Key> L;
  std::map<Key, double> gam;
  for (int i = 0; i < n_leaf; ++i) {
    const Key k = {leaves[4 * i], leaves[4 * i + 1], leaves[4 * i + 2], leaves[4 * i + 3]};
    L.insert(k);
    gam[k] = gamma[i];
  }
  const int v = validate(F, L, n_leaf);
  if (v != MG_OK) return v;
  // When the balance would have to refine a frozen block, bar the parent of the
  // leaf that needs it from refinement and restart from the input (reading A2).
  std::set<Key> forbidden, res;
  int32_t suppressed = 0;
  for (;;) {
    Key bad{};
    if (adapt_once(F, L, gam, eps_r, eps_c, max_level, forbidden, res, bad, suppressed)) break;
    // no progress: the conflicting block is already barred (cannot happen on valid input)
    if (!forbidden.insert(bad).second) return MG_ERR_LAYOUT_2TO1;
  }
  *n_out = (int32_t)res.size();
  if (n_suppressed) *n_suppressed = suppressed;
  if ((int64_t)res.size() > (int64_t)out_capacity || (!out_leaves && !res.empty())) return MG_ERR_ARG;
  int i = 0;
  for (const Key& k : res) {
    for (int t = 0; t < 4; ++t) out_leaves[4 * i + t] = k[t];
    ++i;
  }
  return MG_OK;
}
