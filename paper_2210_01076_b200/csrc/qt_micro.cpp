// qt_micro.cpp -- lean-kernel layer-word lowering (see qt_micro.hpp).
#include "qt_micro.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace qtb {

namespace {

constexpr double kPi = 3.14159265358979323846;
// largest shear factor |tan(phi/2)| accepted for a table entry (|phi| <=
// ~0.94 pi); beyond it the table stays complex multiplies
constexpr double kMaxShear = 12.0;
// carried-scalar magnitude below which the stored state is renormalised
// (the state then holds amplitudes up to 2^300: far from FP64 overflow)
constexpr double kRescaleBelow = 0x1p-300;

bool is_layer_lean(const DOp& d) {
  const uint32_t type = (d.hdr & kOpVariantMask) >> 10;
  if (type == D_XPERM) return (d.hdr & (kOpDl | kOpDg)) == 0;
  if (type == D_DIAG || type == D_PHASE1) return true;  // lowered to M_TDIAG words
  return type == D_LAYER && (d.hdr & kOpFlagMask) == 0;
}

double bits_as_double(uint64_t w) {
  double d;
  std::memcpy(&d, &w, 8);
  return d;
}

// A table's place in the lowered plan, for the final scalar fold.
struct TableRef {
  size_t pass = 0, word = 0, pool = 0;
  std::vector<cplx> phases;  // the table's centred entries
};

// Centres the angles of a table's entries: returns
// false (keep complex multiplies) when an entry is not a unit phase or the
// centred angles need shear factors above kMaxShear.
bool centre_tables(std::vector<cplx>& t, cplx& removed) {
  const size_t n = t.size();
  std::vector<double> ang(n);
  for (size_t s = 0; s < n; ++s) {
    const double r = std::hypot(t[s].re, t[s].im);
    if (!(std::fabs(r - 1.0) <= 1e-12)) return false;
    ang[s] = std::atan2(t[s].im, t[s].re);
  }
  std::vector<double> srt(ang);
  std::sort(srt.begin(), srt.end());
  // largest circular gap between consecutive angles
  double best = srt.front() + 2.0 * kPi - srt.back(), mid = srt.back() + 0.5 * best;
  for (size_t s = 1; s < n; ++s) {
    const double gap = srt[s] - srt[s - 1];
    if (gap > best) {
      best = gap;
      mid = srt[s - 1] + 0.5 * gap;
    }
  }
  if (std::tan(0.5 * (kPi - 0.5 * best)) > kMaxShear) return false;
  const double gamma = mid + kPi;  // opposite the gap's middle
  removed = cplx{std::cos(gamma), std::sin(gamma)};
  const cplx inv{removed.re, -removed.im};
  for (size_t s = 0; s < n; ++s) t[s] = cmul(t[s], inv);
  return true;
}

void push_shear(std::vector<double>& pool, const cplx& t) {
  // e^{i phi}: re += a im; im += b re; re += a im, a = -tan(phi/2), b = sin(phi)
  const double phi = std::atan2(t.im, t.re);
  pool.push_back(-std::tan(0.5 * phi));
  pool.push_back(std::sin(phi));
}

// A rotation [[c, -s], [s, c]] (the round compiler's (c, s), c >= 0),
// lowered to two FMAs per real pair instead of three shears:
//   c >= |s|: c [[1, -t], [t, 1]], t = s / c:  x' = x - t y,  y' = y + t x
//   else:     s [[u, -1], [1, u]], u = c / s:  x' = u x - y,  y' = x + u y
// (|t|, |u| <= 1: each output is one FMA of a perfectly conditioned step).
// The scale factor is uniform over the state, so it is carried like the
// table phases and folded into the plan's last table. Pool: (t, 0) or (u, 1).
void push_rotation(std::vector<double>& pool, double c, double s, cplx& carried) {
  if (c >= std::fabs(s)) {
    pool.push_back(s / c);
    pool.push_back(0.0);
    carried = cplx{carried.re * c, carried.im * c};
  } else {
    pool.push_back(c / s);
    pool.push_back(1.0);
    carried = cplx{carried.re * s, carried.im * s};
  }
}

void pad_even(std::vector<double>& pool) {
  if (pool.size() & 1) pool.push_back(0.0);
}

}  // namespace

bool pass_is_lean(const PlanPass& ps) {
  if (ps.kind != PlanPass::Tile) return false;
  for (const PlanRound& pr : ps.rounds)
    for (const DOp& d : pr.enc.ops)
      if (!is_layer_lean(d)) return false;
  return true;
}

std::vector<MicroPass> lower_plan_micro(const Plan& plan, int reg_bits, const MicroLimits& lim) {
  std::vector<MicroPass> out(plan.passes.size());
  cplx carried{1.0, 0.0};
  TableRef last;
  bool have_last = false;
  for (size_t pi = 0; pi < plan.passes.size(); ++pi) {
    const PlanPass& ps = plan.passes[pi];
    if (!pass_is_lean(ps)) continue;
    const int R = std::min<int>(reg_bits, static_cast<int>(ps.tile_phys.size()));
    const int NS = 1 << R;
    MicroPass& mp = out[pi];
    std::vector<double>& P = mp.pool;
    bool ok = true;
    cplx pass_carried = carried;
    TableRef pass_last = last;
    bool pass_have_last = have_last;
    for (const PlanRound& pr : ps.rounds) {
      if (static_cast<int>(pr.reg.size()) != R) {
        ok = false;
        break;
      }
      mp.round_first.push_back(static_cast<uint16_t>(mp.size()));
      for (const DOp& d : pr.enc.ops) {
        const uint32_t type = (d.hdr & kOpVariantMask) >> 10;
        const double* src = pr.enc.pool.data();
        pad_even(P);
        const uint32_t off = static_cast<uint32_t>(P.size());
        if (type == D_XPERM) {
          P.push_back(bits_as_double(d.lmask));
          P.push_back(bits_as_double(d.gmask));
          mp.words.push_back(off | M_PERM);
          mp.words.push_back(d.hdr);
          continue;
        }
        if (type == D_DIAG || type == D_PHASE1) {
          const uint32_t v = d.hdr & kOpVariantMask;
          const int cs = static_cast<int>((v >> 3) & 7u) - 1;
          const int ds = static_cast<int>(v & 7u) - 1;
          uint32_t smask = 0;
          for (int sl = 0; sl < NS; ++sl)
            if (cs < 0 || ((sl >> cs) & 1)) smask |= 1u << sl;
          P.push_back(bits_as_double(d.lmask));
          P.push_back(bits_as_double(d.dl));
          P.push_back(bits_as_double(d.gmask));
          P.push_back(bits_as_double(d.dg));
          const size_t o = d.arg;
          P.push_back(src[o]);      // d0 = m00
          P.push_back(src[o + 1]);
          P.push_back(src[o + 6]);  // d1 = m11
          P.push_back(src[o + 7]);
          mp.words.push_back(off | M_TDIAG);
          mp.words.push_back(smask | (static_cast<uint32_t>(ds + 1) << 16) |
                             (type == D_PHASE1 ? M_TD_PHASE1 : 0u));
          continue;
        }
        // D_LAYER pool: [table 2 NS][terms 2 nt][rotations 2 each][2x2s 8 each]
        size_t o = d.arg & 0xffffu;
        const uint32_t nt = d.arg >> 16;
        bool tab = (d.hdr & kOpTable) != 0;
        std::vector<cplx> t;
        if (tab) {
          t.resize(NS);
          for (int s = 0; s < NS; ++s) t[s] = cplx{src[o + 2 * s], src[o + 2 * s + 1]};
          o += 2 * NS;
        }
        std::vector<SignTerm> gterms, lterms;
        for (uint32_t k = 0; k < nt; ++k) {
          uint64_t w0, w1;
          std::memcpy(&w0, &src[o + 2 * k], 8);
          std::memcpy(&w1, &src[o + 2 * k + 1], 8);
          SignTerm st{static_cast<uint32_t>(w0), static_cast<uint32_t>(w0 >> 32), w1};
          (st.lcond == 0 && tab ? gterms : lterms).push_back(st);
        }
        o += 2 * nt;
        uint32_t base = d.dl;
        if (tab) {
          // a table of exact +-1 entries is a set of sign flips (integer ops)
          bool signs_only = true;
          uint32_t neg = 0;
          for (int s = 0; s < NS && signs_only; ++s) {
            signs_only = t[s].im == 0.0 && (t[s].re == 1.0 || t[s].re == -1.0);
            if (t[s].re == -1.0) neg |= 1u << s;
          }
          if (signs_only) {
            base ^= neg;
            tab = false;
            lterms.insert(lterms.end(), gterms.begin(), gterms.end());
            gterms.clear();
          }
        }
        if (static_cast<int>(gterms.size()) > kMaxTableVariantTerms) {
          lterms.insert(lterms.end(), gterms.begin(), gterms.end());
          gterms.clear();
        }
        uint32_t x = off;
        // A partial table keeps its identity entries. The round compiler's
        // tables carry the phases in front of the layer's rotations: a layer
        // with m of R slots rotating has exact ones on the 2^(R-m) slots whose
        // rotating bits are all 0 (C3: 150 of 232 tables). Identity entries
        // cost nothing in the compiled kernels, so such a table is not centred
        // (that would turn the ones into a common phase) and the sign flips
        // are not folded into it; entries beyond a quarter turn give their -1
        // to the flip mask instead, so every shear factor stays <= 1
        // (C3: 1864 -> 1736 FP64 ops per amplitude). QTB_PARTIAL_TABLES=0:
        // every table centred as a whole.
        int n_ident = 0;
        bool unit = tab;
        for (int s = 0; tab && s < NS; ++s) {
          n_ident += (t[s].re == 1.0 && t[s].im == 0.0) ? 1 : 0;
          unit = unit && std::fabs(std::hypot(t[s].re, t[s].im) - 1.0) <= 1e-12;
        }
        static const bool partial_on = [] {
          const char* e = std::getenv("QTB_PARTIAL_TABLES");
          return !e || std::atoi(e) != 0;
        }();
        bool partial = partial_on && tab && unit && n_ident >= 2 && n_ident < NS;
        if (partial_on && tab && unit && n_ident == 0) {
          // a full table of unit phases: its slot-0 phase is a scalar of the
          // whole state (carried like the centring phases), which leaves an
          // exact 1 on slot 0 -- one entry less to apply
          const double phi0 = std::atan2(t[0].im, t[0].re);
          const cplx ph{std::cos(phi0), std::sin(phi0)};  // the phase only (like centre_tables)
          const cplx inv{ph.re, -ph.im};
          pass_carried = cmul(pass_carried, ph);
          for (int s = NS - 1; s >= 0; --s) t[s] = s == 0 ? cplx{1.0, 0.0} : cmul(t[s], inv);
          n_ident = 1;
          for (int s = 1; s < NS; ++s) n_ident += (t[s].re == 1.0 && t[s].im == 0.0) ? 1 : 0;
          partial = n_ident < NS || !gterms.empty();
          if (!partial) {  // it was a pure scalar: no table at all
            tab = false;
          }
        }
        if (partial) {
          const size_t nv = gterms.size();
          for (const SignTerm& g : gterms) {
            P.push_back(bits_as_double(g.gcond));
            P.push_back(bits_as_double(g.slots));
          }
          const size_t toff = P.size();
          for (int s = 0; s < NS; ++s) {
            if (t[s].re == 1.0 && t[s].im == 0.0) {
              P.push_back(0.0);
              P.push_back(0.0);
              continue;
            }
            if (t[s].re < 0.0) {  // |phi| > pi/2: -1 to the flips
              t[s] = cplx{-t[s].re, -t[s].im};
              base ^= 1u << s;
            }
            push_shear(P, t[s]);
          }
          pass_last = TableRef{pi, mp.words.size(), toff, t};
          pass_have_last = true;
          x |= M_STAB | (static_cast<uint32_t>(nv) << M_NV_SHIFT);
        } else if (tab) {
          // unconditional flips join the table; each tile-uniform term
          // becomes (condition, slot mask): the table's output is negated on
          // those slots when the tile's global bits meet the condition
          for (int s = 0; s < NS; ++s)
            if ((base >> s) & 1u) t[s] = cplx{-t[s].re, -t[s].im};
          base = 0;
          const size_t nv = gterms.size();
          for (const SignTerm& g : gterms) {
            P.push_back(bits_as_double(g.gcond));
            P.push_back(bits_as_double(g.slots));
          }
          const size_t toff = P.size();
          bool scalar = nv == 0;
          for (int s = 1; s < NS && scalar; ++s)
            scalar = t[s].re == t[0].re && t[s].im == t[0].im;
          cplx removed;
          if (scalar) {
            // a pure scalar: carried, no table at all
            pass_carried = cmul(pass_carried, t[0]);
            P.resize(off);
          } else if (centre_tables(t, removed)) {
            pass_carried = cmul(pass_carried, removed);
            for (const cplx& c : t) push_shear(P, c);
            pass_last = TableRef{pi, mp.words.size(), toff, t};
            pass_have_last = true;
            x |= M_STAB | (static_cast<uint32_t>(nv) << M_NV_SHIFT);
          } else {
            for (const cplx& c : t) {
              P.push_back(c.re);
              P.push_back(c.im);
            }
            x |= M_CTAB | (static_cast<uint32_t>(nv) << M_NV_SHIFT);
          }
        }
        uint32_t y = 0;
        if (base || !lterms.empty()) {
          if (lterms.size() > 0xffffu) {
            ok = false;
            break;
          }
          for (const SignTerm& st : lterms) {
            const uint64_t w0 = static_cast<uint64_t>(st.slots) |
                                (static_cast<uint64_t>(st.lcond) << 32);
            P.push_back(bits_as_double(w0));
            P.push_back(bits_as_double(st.gcond));
          }
          x |= M_SIGN;
          y = base | (static_cast<uint32_t>(lterms.size()) << 16);
        }
        const uint32_t rmask = (d.hdr >> 6) & 15u;
        for (int a = 0; a < R; ++a) {
          if (!(rmask & (1u << a))) continue;
          // the round compiler's rotation (c, s), |theta| <= pi/2, becomes a
          // scaled rotation of two FMAs per real pair; its scale (c or s)
          // joins the carried scalar (see push_rotation)
          push_rotation(P, src[o], src[o + 1], pass_carried);
          o += 2;
        }
        for (int a = 0; a < R; ++a) {
          if (!(d.lmask & (1u << a))) continue;
          for (int k = 0; k < 8; ++k) P.push_back(src[o + k]);
          o += 8;
        }
        x |= (rmask << M_ROT_SHIFT) | ((d.lmask & 15u) << M_DENSE_SHIFT);
        if ((x & ~0xffffu) == 0) {
          P.resize(off);  // nothing left (a scalar table)
          continue;
        }
        mp.words.push_back(x);
        mp.words.push_back(y);
        // the scaled rotations grow the stored state by up to sqrt(2) each:
        // long before it could overflow, an exact power-of-two scale word
        // (a complex table of 2^-m) renormalises it
        const double mag = std::hypot(pass_carried.re, pass_carried.im);
        if (mag > 0.0 && mag < kRescaleBelow) {
          const double f = std::ldexp(1.0, std::ilogb(mag));
          pad_even(P);
          const uint32_t so = static_cast<uint32_t>(P.size());
          for (int s = 0; s < NS; ++s) {
            P.push_back(f);
            P.push_back(0.0);
          }
          pass_carried = cplx{pass_carried.re / f, pass_carried.im / f};
          mp.words.push_back(so | M_CTAB);
          mp.words.push_back(0);
        }
      }
      if (!ok) break;
      if (mp.size() == mp.round_first.back()) {  // an empty round: one no-op word
        mp.words.push_back(0);
        mp.words.push_back(0);
      }
      mp.words[mp.words.size() - 2] |= M_LAST;
      mp.round_count.push_back(
          static_cast<uint16_t>(mp.size() - mp.round_first.back()));
    }
    if (!ok || P.size() > std::min<size_t>(0xffffu, lim.pool) || mp.size() > lim.ops ||
        ps.rounds.size() > lim.rounds) {
      out[pi] = MicroPass{};  // the generic kernel runs this pass
      continue;
    }
    mp.ok = true;
    carried = pass_carried;
    last = std::move(pass_last);
    have_last = pass_have_last;
  }
  if (carried.re == 1.0 && carried.im == 0.0) return out;
  if (have_last) {
    // the plan's last shear table absorbs every removed scalar: it becomes
    // complex multiplies with the scalar folded in
    MicroPass& mp = out[last.pass];
    mp.words[last.word] = (mp.words[last.word] & ~M_STAB) | M_CTAB;
    for (size_t s = 0; s < last.phases.size(); ++s) {
      const cplx c = cmul(last.phases[s], carried);
      mp.pool[last.pool + 2 * s] = c.re;
      mp.pool[last.pool + 2 * s + 1] = c.im;
    }
    return out;
  }
  // only scalar tables were seen: one complex table of the scalar joins the
  // last lowered round
  for (size_t pi = out.size(); pi-- > 0;) {
    MicroPass& mp = out[pi];
    if (!mp.ok || mp.round_count.empty()) continue;
    const int R = std::min<int>(reg_bits, static_cast<int>(plan.passes[pi].tile_phys.size()));
    pad_even(mp.pool);
    const uint32_t off = static_cast<uint32_t>(mp.pool.size());
    for (int s = 0; s < (1 << R); ++s) {
      mp.pool.push_back(carried.re);
      mp.pool.push_back(carried.im);
    }
    mp.words[mp.words.size() - 2] &= ~M_LAST;
    mp.words.push_back(off | M_CTAB | M_LAST);
    mp.words.push_back(0);
    mp.round_count.back() += 1;
    return out;
  }
  return out;
}

double micro_fp64_per_amp(const MicroPass& mp, int R) {
  const int NS = 1 << R;
  double fp = 0.0;
  for (size_t w = 0; w < mp.size(); ++w) {
    const uint32_t x = mp.words[2 * w], y = mp.words[2 * w + 1];
    if (x & M_PERM) continue;
    if (x & M_TDIAG) {
      fp += 4.0 * __builtin_popcount(y & 0xffffu) / NS;
      continue;
    }
    uint32_t off = x & 0xffffu;
    if (x & (M_STAB | M_CTAB)) {
      const uint32_t nv = (x >> M_NV_SHIFT) & 3u;
      off += 2 * nv;
      int live = 0;
      for (int s = 0; s < NS; ++s) {
        const double a = mp.pool[off + 2 * s], b = mp.pool[off + 2 * s + 1];
        const bool ident = (x & M_STAB) ? (a == 0.0 && b == 0.0) : (a == 1.0 && b == 0.0);
        live += ident ? 0 : 1;
      }
      fp += ((x & M_STAB) ? 3.0 : 4.0) * live / NS;
    }
    fp += 2.0 * __builtin_popcount((x >> M_ROT_SHIFT) & 15u) +
          8.0 * __builtin_popcount((x >> M_DENSE_SHIFT) & 15u);
  }
  return fp;
}

}  // namespace qtb
