// Offline template inference (the reference's analyzer.py:185-441), native.
//
// Host C++ (no device code): per kernel of a task, identify pointer
// arguments, fit each pointer's access family as fixed / linear in a product
// of <= 3 integer slots / strided, and measure the fraction of observed
// regions the rules do not cover.  Exactly the matching order of
// paper_2512_24637_b200/analyzer.py (which mirrors the reference):
//   pointer args = 64-bit args equal to a region start in every record;
//   constant-offset args = smallest c with arg+c a region start below 2*arg;
//   candidate slots sorted by slot rank, positive in every record, deduplicated
//   by value signature; fits tried by (fewest factors, lowest slots).
// Ratio equality v_r / P_r == v_0 / P_0 is decided exactly with 256-bit cross
// products (values and slot values < 2^64).  A kernel whose numbers fall
// outside that range is reported back (status 1) and the host analyzer does
// it.  The coefficient itself (v_0 / P_0, a reduced fraction) is formed by the
// host from the first record, so no big-number division is needed here.
#include "msched_internal.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <vector>

namespace {

typedef __int128 i128;
typedef unsigned __int128 u128;

struct Region { int64_t a, len; };        // [a, a + len)
struct Rec {
  const msg_cmd* cmd;
  std::vector<Region> regs;                 // coalesced observed regions
  double lat;
};

struct Slot {                               // one named slot value of one record
  int64_t code;                             // _abi.slot_code of the name
  std::tuple<int, int64_t, int, int64_t, int> rank;
  i128 value;
};

i128 arg_value(const msg_arg& a) { return (i128)(((u128)(uint64_t)a.hi << 64) | (u128)a.lo); }
bool plain64(const msg_arg& a) { return a.raw_len < 0 && a.width == 64; }

// analyzer.py:75-85 slot_values; codes as in _abi.slot_code
std::vector<Slot> slot_values(const Rec& r, const msg_arg* args, const uint8_t* blob) {
  std::vector<Slot> out;
  const msg_cmd& c = *r.cmd;
  for (int i = 0; i < c.nargs; ++i) {
    const msg_arg& a = args[c.arg_off + i];
    if (a.raw_len < 0) {
      out.push_back({(int64_t)i << 2, {0, i, 0, 0, 0}, arg_value(a)});
    } else {
      const uint8_t* raw = blob + a.raw_off;
      for (int64_t o = 0; o + 8 <= a.raw_len; o += 8) {
        uint64_t v; std::memcpy(&v, raw + o, 8);
        out.push_back({1 | ((int64_t)i << 2) | (o << 18) | (1ll << 50), {0, i, 1, o, -64}, (i128)v});
      }
      for (int64_t o = 0; o + 4 <= a.raw_len; o += 4) {
        uint32_t v; std::memcpy(&v, raw + o, 4);
        out.push_back({1 | ((int64_t)i << 2) | (o << 18), {0, i, 1, o, -32}, (i128)v});
      }
    }
  }
  for (int d = 0; d < 6; ++d) out.push_back({2 | ((int64_t)d << 2), {1, d, 0, 0, 0}, (i128)c.dims[d]});
  return out;
}

struct U256 { uint64_t w[4]; };
U256 mul4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  uint64_t r[4] = {a, 0, 0, 0};
  const uint64_t f[3] = {b, c, d};
  for (uint64_t m : f) {
    u128 carry = 0;
    for (int k = 0; k < 4; ++k) {
      u128 x = (u128)r[k] * m + carry;
      r[k] = (uint64_t)x;
      carry = x >> 64;
    }
  }
  U256 o; std::memcpy(o.w, r, sizeof(r));
  return o;
}
bool eq(const U256& x, const U256& y) { return std::memcmp(x.w, y.w, sizeof(x.w)) == 0; }

struct Expr { int nslots = 0; int64_t slot[3] = {0, 0, 0}; int64_t v0 = 0; bool ok = false; };

struct Fitter {
  const std::vector<Rec>& recs;
  std::vector<std::vector<Slot>> tables;
  std::vector<std::vector<uint64_t>> cand;   // candidate slot values per record
  std::vector<int64_t> cand_code;
  bool overflow = false;

  Fitter(const std::vector<Rec>& r, const msg_arg* args, const uint8_t* blob) : recs(r) {
    for (auto& x : recs) tables.push_back(slot_values(x, args, blob));
  }
  // analyzer.py _Fitter.factor_slots
  void factor_slots(const std::set<int>& ptr_idx) {
    cand.clear(); cand_code.clear();
    std::vector<Slot> names = tables[0];
    std::stable_sort(names.begin(), names.end(), [](const Slot& a, const Slot& b) { return a.rank < b.rank; });
    std::set<std::vector<i128>> sigs;
    for (auto& s : names) {
      int kind = (int)(s.code & 3);
      if (kind == 0 && ptr_idx.count((int)((s.code >> 2) & 0xffff))) continue;
      std::vector<i128> sig;
      bool bad = false;
      for (auto& t : tables) {
        auto it = std::find_if(t.begin(), t.end(), [&](const Slot& x) { return x.code == s.code; });
        if (it == t.end() || it->value <= 0) { bad = true; break; }
        sig.push_back(it->value);
      }
      if (bad || sigs.count(sig)) continue;
      sigs.insert(sig);
      std::vector<uint64_t> v;
      for (i128 x : sig) {
        if (x >= ((i128)1 << 64)) overflow = true;   // beyond the 256-bit cross products
        v.push_back((uint64_t)x);
      }
      cand.push_back(v);
      cand_code.push_back(s.code);
    }
  }
  // analyzer.py _Fitter.fit: constant, else first exact coeff*prod by (fewest factors, lowest slots)
  Expr fit(const std::vector<int64_t>& vals) {
    Expr e;
    bool same = true;
    for (auto v : vals) same = same && v == vals[0];
    if (same) { e.ok = true; e.v0 = vals[0]; return e; }
    for (auto v : vals)
      if (v <= 0) { overflow = true; return e; }     // host handles non-positive values
    const int n = (int)cand.size(), R = (int)vals.size();
    int idx[3];
    for (int k = 1; k <= 3; ++k) {
      for (int j = 0; j < k; ++j) idx[j] = 0;
      while (true) {
        auto prod_at = [&](int r) {
          uint64_t f[3] = {1, 1, 1};
          for (int j = 0; j < k; ++j) f[j] = cand[idx[j]][r];
          return mul4((uint64_t)vals[0], f[0], f[1], f[2]);   // v_0 * P_r
        };
        uint64_t g[3] = {1, 1, 1};
        for (int j = 0; j < k; ++j) g[j] = cand[idx[j]][0];
        bool all = true;
        for (int r = 1; r < R && all; ++r) {
          U256 lhs = mul4((uint64_t)vals[r], g[0], g[1], g[2]);   // v_r * P_0
          all = eq(lhs, prod_at(r));
        }
        if (all) {   // coefficient v_0 / P_0 > 0
          e.ok = true; e.nslots = k; e.v0 = vals[0];
          for (int j = 0; j < k; ++j) e.slot[j] = cand_code[idx[j]];
          return e;
        }
        // next combination with replacement (non-decreasing indices)
        int p = k - 1;
        while (p >= 0 && idx[p] == n - 1) --p;
        if (p < 0 || n == 0) break;
        ++idx[p];
        for (int j = p + 1; j < k; ++j) idx[j] = idx[p];
      }
    }
    return e;
  }
};

struct Rule {
  int ptr; int64_t off; int kind;           // 0 fixed 1 linear 2 strided 3 unpredictable
  Expr e[3];
  // per record: base and the family values the rule reproduces for it
  std::vector<i128> base;
  std::vector<int64_t> size, stride, chunk, count;
};

// analyzer.py infer_rule
Rule infer_rule(const std::vector<Rec>& recs, const msg_arg* args, int i, int64_t o,
                const std::vector<std::pair<int, int64_t>>& ptrs, Fitter& F) {
  Rule dead{i, o, 3, {}, {}, {}, {}, {}, {}};
  std::vector<std::vector<Region>> fams;
  std::vector<i128> bases;
  for (auto& r : recs) {
    const msg_cmd& c = *r.cmd;
    i128 base = arg_value(args[c.arg_off + i]) + o;
    bool have = false;
    i128 ceiling = 0;
    for (auto& p : ptrs) {
      if (p.first == i && p.second == o) continue;
      i128 b = arg_value(args[c.arg_off + p.first]) + p.second;
      if (b > base && (!have || b < ceiling)) { ceiling = b; have = true; }
    }
    std::vector<Region> fam;
    for (auto& g : r.regs)
      if ((i128)g.a >= base && (!have || (i128)g.a < ceiling)) fam.push_back(g);
    if (fam.empty() || (i128)fam[0].a != base) return dead;
    fams.push_back(fam);
    bases.push_back(base);
  }
  std::set<int> pidx;
  for (auto& p : ptrs) pidx.insert(p.first);
  F.factor_slots(pidx);
  Rule out{i, o, 0, {}, bases, {}, {}, {}, {}};
  bool single = true;
  for (auto& f : fams) single = single && f.size() == 1;
  if (single) {
    for (auto& f : fams) out.size.push_back(f[0].len);
    bool same = true;
    for (auto v : out.size) same = same && v == out.size[0];
    if (same) { out.kind = 0; out.e[0].ok = true; out.e[0].v0 = out.size[0]; return out; }
    Expr e = F.fit(out.size);
    if (!e.ok || e.nslots == 0) return dead;
    out.kind = 1; out.e[0] = e;
    return out;
  }
  for (auto& f : fams) {
    if (f.size() < 2) return dead;
    std::set<int64_t> st, ln;
    for (size_t k = 0; k + 1 < f.size(); ++k) st.insert(f[k + 1].a - f[k].a);
    for (auto& g : f) ln.insert(g.len);
    if (st.size() != 1 || ln.size() != 1) return dead;
    out.stride.push_back(*st.begin());
    out.chunk.push_back(*ln.begin());
    out.count.push_back((int64_t)f.size());
  }
  Expr es = F.fit(out.stride), ec = F.fit(out.chunk), en = F.fit(out.count);
  if (!es.ok || !ec.ok || !en.ok) return dead;
  out.kind = 2; out.e[0] = es; out.e[1] = ec; out.e[2] = en;
  return out;
}

bool covered(const std::vector<std::pair<i128, i128>>& regs, const Region& g) {
  for (auto& p : regs)
    if (p.first <= (i128)g.a && p.second >= (i128)g.a + g.len) return true;
  return false;
}

}  // namespace

extern "C" int msg_analyze(const msg_cmd* cmds, int32_t ncmd, const msg_arg* args, const uint8_t* blob,
                           int64_t blob_len, const msg_range* gt, const double* latency, int32_t nkernels,
                           int32_t* status, double* latency_out, double* unpred_out, msg_arule* rules_out,
                           int32_t rules_cap, int32_t* rule_off) {
  (void)blob_len;
  if (ncmd < 0 || nkernels < 0 || (nkernels && (!status || !latency_out || !unpred_out || !rule_off)))
    return MSG_E_INVAL;
  try {
    std::vector<std::vector<Rec>> by(nkernels);
    for (int32_t i = 0; i < ncmd; ++i) {
      const msg_cmd& c = cmds[i];
      if (c.kind != MSG_CMD_KERNEL) continue;
      if (c.kernel < 0 || c.kernel >= nkernels) return MSG_E_INVAL;
      Rec r{&c, {}, latency[i]};
      // coalesce_regions: sort by start (stable), merge strictly overlapping
      std::vector<Region> g;
      for (int k = 0; k < c.ngt; ++k) g.push_back({gt[c.gt_off + k].start, gt[c.gt_off + k].len});
      std::stable_sort(g.begin(), g.end(), [](const Region& x, const Region& y) { return x.a < y.a; });
      for (auto& x : g) {
        if (!r.regs.empty() && x.a < r.regs.back().a + r.regs.back().len) {
          Region& top = r.regs.back();
          int64_t end = std::max(top.a + top.len, x.a + x.len);
          top.len = end - top.a;
        } else {
          r.regs.push_back(x);
        }
      }
      by[c.kernel].push_back(std::move(r));
    }
    int32_t nr = 0;
    for (int32_t k = 0; k < nkernels; ++k) {
      rule_off[k] = nr;
      status[k] = 0;
      auto& recs = by[k];
      if (recs.empty()) { status[k] = 1; continue; }
      const int nargs0 = recs[0].cmd->nargs;
      // identify_pointer_args
      std::vector<std::pair<int, int64_t>> ptrs;
      for (int i = 0; i < nargs0; ++i) {
        bool all = true;
        for (auto& r : recs) {
          const msg_cmd& c = *r.cmd;
          if (i >= c.nargs || !plain64(args[c.arg_off + i])) { all = false; break; }
          i128 v = arg_value(args[c.arg_off + i]);
          bool hit = false;
          for (auto& g : r.regs) hit = hit || (i128)g.a == v;
          if (!hit) { all = false; break; }
        }
        if (all) ptrs.push_back({i, 0});
      }
      // _constant_offset for the other args (the host raises on ragged arg counts)
      bool ragged = false;
      for (int i = 0; i < nargs0 && !ragged; ++i) {
        bool isp = false;
        for (auto& p : ptrs) isp = isp || p.first == i;
        if (isp) continue;
        std::set<i128> common;
        bool first = true, none = false;
        for (auto& r : recs) {
          const msg_cmd& c = *r.cmd;
          if (i >= c.nargs) { ragged = true; break; }
          const msg_arg& a = args[c.arg_off + i];
          if (!plain64(a)) { none = true; break; }
          i128 v = arg_value(a);
          std::set<i128> here;
          for (auto& g : r.regs)
            if (v < (i128)g.a && (i128)g.a < 2 * v) here.insert((i128)g.a - v);
          if (first) { common = here; first = false; }
          else {
            std::set<i128> x;
            std::set_intersection(common.begin(), common.end(), here.begin(), here.end(), std::inserter(x, x.begin()));
            common.swap(x);
          }
          if (common.empty()) { none = true; break; }
        }
        if (!ragged && !none && !common.empty()) ptrs.push_back({i, (int64_t)*common.begin()});
      }
      if (ragged) { status[k] = 1; continue; }
      // records with ragged argument counts past the pointer args: host path
      for (auto& r : recs)
        for (auto& p : ptrs)
          if (p.first >= r.cmd->nargs) ragged = true;
      if (ragged) { status[k] = 1; continue; }
      std::sort(ptrs.begin(), ptrs.end());
      Fitter F(recs, args, blob);
      std::vector<Rule> rules;
      for (auto& p : ptrs) rules.push_back(infer_rule(recs, args, p.first, p.second, ptrs, F));
      if (F.overflow) { status[k] = 1; continue; }
      // latency: mean in record order, summed the way CPython >= 3.12's
      // sum() adds floats (Neumaier compensation), so the host's descriptor
      // floats come out bit for bit
      double s = 0.0, comp = 0.0;
      for (auto& r : recs) {
        double t = s + r.lat;
        if (std::fabs(s) >= std::fabs(r.lat)) comp += (s - t) + r.lat;
        else comp += (r.lat - t) + s;
        s = t;
      }
      if (comp != 0.0 && std::isfinite(comp)) s += comp;
      latency_out[k] = s / (double)recs.size();
      // uncovered fraction: the rules reproduce each record's own family
      int64_t total = 0, misses = 0;
      for (size_t ri = 0; ri < recs.size(); ++ri) {
        std::vector<std::pair<i128, i128>> regs;
        for (auto& ru : rules) {
          if (ru.kind == 3) continue;
          i128 b = ru.base[ri];
          if (ru.kind == 0 || ru.kind == 1) {
            int64_t n = ru.kind == 0 ? ru.e[0].v0 : ru.size[ri];
            regs.push_back({b, b + std::max<int64_t>(n, 1)});
          } else {
            int64_t st = ru.stride[ri], ch = std::max<int64_t>(ru.chunk[ri], 1), ct = ru.count[ri];
            for (int64_t j = 0; j < ct; ++j) regs.push_back({b + (i128)j * st, b + (i128)j * st + ch});
          }
        }
        for (auto& g : recs[ri].regs) {
          ++total;
          misses += !covered(regs, g);
        }
      }
      unpred_out[k] = total ? (double)misses / (double)total : 0.0;
      for (auto& ru : rules) {
        if (ru.kind == 3) continue;
        if (rules_out && nr < rules_cap) {
          msg_arule& o = rules_out[nr];
          std::memset(&o, 0, sizeof(o));
          o.ptr_arg = ru.ptr; o.offset = ru.off; o.kind = ru.kind;
          for (int q = 0; q < 3; ++q) {
            o.nslots[q] = ru.e[q].nslots;
            o.v0[q] = ru.e[q].v0;
            for (int j = 0; j < 3; ++j) o.slot[q][j] = ru.e[q].slot[j];
          }
        }
        ++nr;
      }
    }
    if (nkernels) rule_off[nkernels] = nr;
    return nr > rules_cap ? MSG_E_INVAL : MSG_OK;
  } catch (const std::exception&) {
    return MSG_E_OOM;
  }
}
