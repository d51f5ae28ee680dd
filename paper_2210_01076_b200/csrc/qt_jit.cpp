// qt_jit.cpp -- compiled tile passes: source generation, NVRTC, cache.
#include "qt_jit.hpp"

#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <array>
#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <future>
#include <memory>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <thread>

#include <pthread.h>
#include <dirent.h>
#include <sys/stat.h>
#include <sys/types.h>
#include <unistd.h>
#include <unordered_map>

#include "qt_gates.hpp"

namespace qtb {

namespace {

// ---------------------------------------------------------------------------
// Device prelude of every compiled pass (NVRTC has no standard headers).
// The bodies mirror qt_tilepass.cu; in straight-line code register swaps are
// plain renames, so no XOR-swap tricks are needed.
// ---------------------------------------------------------------------------
const char* kPrelude = R"PRE(
typedef unsigned int u32;
typedef unsigned long long u64;
#define FI __device__ __forceinline__
FI u64 pdep64(u64 x, u64 mask) {
  u64 r = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    if (!mask) break;
    const u64 low = mask & (~mask + 1);
    if (x & 1) r |= low;
    x >>= 1;
    mask ^= low;
  }
  return r;
}
FI u32 swz(u32 j) { return j ^ ((j >> 3) & 7u) ^ ((j >> 6) & 7u) ^ ((j >> 9) & 7u) ^ ((j >> 12) & 7u); }
FI u32 insert_zero(u32 x, u32 p) { return ((x >> p) << (p + 1)) | (x & ((1u << p) - 1u)); }
FI bool finite2(double2 v) {
  const u32 hx = __double2hiint(v.x), hy = __double2hiint(v.y);
  return ((hx & 0x7ff00000u) != 0x7ff00000u) && ((hy & 0x7ff00000u) != 0x7ff00000u);
}
// x += a y; y += b x; x += a y on the pair (v[s], v[s1])
FI void shear(double2& x, double2& y, double a, double b) {
  x.x = fma(a, y.x, x.x); x.y = fma(a, y.y, x.y);
  y.x = fma(b, x.x, y.x); y.y = fma(b, x.y, y.y);
  x.x = fma(a, y.x, x.x); x.y = fma(a, y.y, x.y);
}
// scaled rotations (qt_micro.cpp push_rotation): c [[1, -t], [t, 1]] and
// s [[u, -1], [1, u]], two FMAs per real pair (same operations as the
// interpreter's pair_srot)
FI void trot(double2& x, double2& y, double k) {
  const double2 a = x, b = y;
  x.x = fma(-k, b.x, a.x); x.y = fma(-k, b.y, a.y);
  y.x = fma(k, a.x, b.x); y.y = fma(k, a.y, b.y);
}
FI void urot(double2& x, double2& y, double k) {
  const double2 a = x, b = y;
  x.x = fma(k, a.x, -b.x); x.y = fma(k, a.y, -b.y);
  y.x = fma(k, b.x, a.x); y.y = fma(k, b.y, a.y);
}
// e^{i phi} on one amplitude as shears of (re, im)
FI void pshear(double2& v, double a, double b) {
  v.x = fma(a, v.y, v.x); v.y = fma(b, v.x, v.y); v.x = fma(a, v.y, v.x);
}
FI void cscale(double2& x, double br, double bi) {
  const double p0 = -bi * x.y, p1 = bi * x.x;
  x.x = fma(br, x.x, p0); x.y = fma(br, x.y, p1);
}
FI void dense(double2& a, double2& b, double m0r, double m0i, double m1r, double m1i,
              double m2r, double m2i, double m3r, double m3i) {
  const double p0 = fma(m1r, b.x, fma(-m1i, b.y, -m0i * a.y));
  const double p1 = fma(m1r, b.y, fma(m1i, b.x, m0i * a.x));
  const double p2 = fma(m2r, a.x, fma(-m2i, a.y, -m3i * b.y));
  const double p3 = fma(m2r, a.y, fma(m2i, a.x, m3i * b.x));
  a.x = fma(m0r, a.x, p0); a.y = fma(m0r, a.y, p1);
  b.x = fma(m3r, b.x, p2); b.y = fma(m3r, b.y, p3);
}
FI void swap2(double2& a, double2& b) { const double2 t = a; a = b; b = t; }
FI void cswap2(double2& a, double2& b, bool c) {
  const double2 x = a, y = b;
  a = c ? y : x; b = c ? x : y;
}
FI double flipd(double d, u32 sg) { return __hiloint2double(__double2hiint(d) ^ sg, __double2loint(d)); }
FI void flip2(double2& v, u32 sg) { v.x = flipd(v.x, sg); v.y = flipd(v.y, sg); }
FI void neg2(double2& v) { flip2(v, 0x80000000u); }
)PRE";

// Exact hexadecimal-float literal of d, formatted from its bits (not with
// printf's %a, whose radix character follows the process locale).
std::string hexd(double d) {
  uint64_t w;
  std::memcpy(&w, &d, 8);
  const bool neg = (w >> 63) != 0;
  const int e = static_cast<int>((w >> 52) & 0x7ffu);
  const uint64_t m = w & ((1ull << 52) - 1);
  if (e == 0x7ff) throw std::runtime_error("non-finite literal");
  char b[48];
  if (e == 0 && m == 0) {
    std::snprintf(b, sizeof(b), "%s0x0p+0", neg ? "-" : "");
  } else {
    const int ex = e == 0 ? -1022 : e - 1023;
    std::snprintf(b, sizeof(b), "%s0x%d.%013llxp%+d", neg ? "-" : "", e == 0 ? 0 : 1,
                  static_cast<unsigned long long>(m), ex);
  }
  return b;
}

std::string hexu(uint64_t x) {
  char b[32];
  std::snprintf(b, sizeof(b), "0x%llxull", static_cast<unsigned long long>(x));
  return b;
}

uint64_t raw_bits(double d) {
  uint64_t w;
  std::memcpy(&w, &d, 8);
  return w;
}

// FP64 constants of a pass, as hex-float literals in the instruction stream.
// (Measured slower on C3 and removed: the constants in a __constant__ array
// read with uniform loads -- the pass's constants overflow the per-SM
// constant cache -- or copied once per CTA into shared memory. Literals ride
// the instruction fetch, two uniform moves per non-encodable double.)
// With a kernel-parameter block (JitPassSpec::kparam) the distinct
// constants go to `K.k[i]` instead: DFMA reads them through uniform loads of
// the parameter bank (one LDCU.128 per two doubles instead of four UMOVs).
struct Consts {
  bool param = false;
  std::vector<double> vals;
  std::unordered_map<uint64_t, int> index;
  std::string operator()(double d) {
    if (!param) return hexd(d);
    uint64_t w;
    std::memcpy(&w, &d, 8);
    auto it = index.find(w);
    if (it == index.end()) {
      it = index.emplace(w, static_cast<int>(vals.size())).first;
      vals.push_back(d);
    }
    return "K.k[" + std::to_string(it->second) + "]";
  }
  std::string pair(double a, double b) { std::string x = (*this)(a); return x + ", " + (*this)(b); }
};
constexpr size_t kMaxKParams = 3800;  // doubles (kernel parameters <= 32764 bytes)

// Code of one layer word.
void emit_word(std::ostringstream& os, Consts& kc, int R, uint32_t x, uint32_t y,
               const std::vector<double>& P) {
  const int NS = 1 << R;
  uint32_t off = x & 0xffffu;
  if (x & M_PERM) {
    const uint32_t a = (y >> 6) & 15u;
    const int cs = static_cast<int>((y >> 3) & 7u) - 1;
    const bool masked = (y & kOpLctl) != 0, gctl = (y & kOpGctl) != 0;
    const uint64_t lm = raw_bits(P[off]) & 0xffffffffull, gm = raw_bits(P[off + 1]);
    os << "  {";
    std::string pre;
    if (gctl) os << " if ((g & " << hexu(gm) << ") == " << hexu(gm) << ")";
    os << " {";
    if (masked) os << " const bool c = (jb & " << lm << "u) == " << lm << "u;";
    for (int s = 0; s < NS; ++s) {
      if (s & (1 << a)) continue;
      if (cs >= 0 && !((s >> cs) & 1)) continue;
      const int s1 = s | (1 << a);
      if (masked) os << " cswap2(v" << s << ", v" << s1 << ", c);";
      else os << " swap2(v" << s << ", v" << s1 << ");";
    }
    os << " } }\n";
    return;
  }
  if (x & M_TDIAG) {
    const uint64_t lm = raw_bits(P[off]) & 0xffffffffull, dl = raw_bits(P[off + 1]) & 0xffffffffull;
    const uint64_t gm = raw_bits(P[off + 2]), dg = raw_bits(P[off + 3]);
    const int ds = static_cast<int>((y >> 16) & 15u) - 1;
    const bool ph1 = (y & M_TD_PHASE1) != 0;
    const std::string d0 = kc(P[off + 4]) + ", " + kc(P[off + 5]), d1 = kc(P[off + 6]) + ", " + kc(P[off + 7]);
    os << "  {";
    std::string cond;
    if (lm) cond += "(jb & " + std::to_string(lm) + "u) == " + std::to_string(lm) + "u";
    if (gm) cond += std::string(cond.empty() ? "" : " && ") + "(g & " + hexu(gm) + ") == " + hexu(gm);
    if (!cond.empty()) os << " if (" << cond << ")";
    os << " {";
    if (ds < 0) {
      std::string tb;
      if (dl) tb += "(jb & " + std::to_string(dl) + "u) != 0";
      if (dg) tb += std::string(tb.empty() ? "" : " || ") + "(g & " + hexu(dg) + ") != 0";
      if (tb.empty()) tb = "false";
      os << " const bool tb = " << tb << ";";
      if (ph1) os << " if (tb) {";
      for (int s = 0; s < NS; ++s) {
        if (!((y >> s) & 1u)) continue;
        if (ph1) os << " cscale(v" << s << ", " << d1 << ");";
        else os << " cscale(v" << s << ", tb ? " << kc(P[off + 6]) << " : " << kc(P[off + 4]) << ", tb ? "
                << kc(P[off + 7]) << " : " << kc(P[off + 5]) << ");";
      }
      if (ph1) os << " }";
    } else {
      for (int s = 0; s < NS; ++s) {
        if (!((y >> s) & 1u)) continue;
        const bool b = ((s >> ds) & 1) != 0;
        if (ph1 && !b) continue;
        os << " cscale(v" << s << ", " << (b ? d1 : d0) << ");";
      }
    }
    os << " } }\n";
    return;
  }
  if (x & (M_STAB | M_CTAB)) {
    const uint32_t nv = (x >> M_NV_SHIFT) & 3u;
    const uint32_t toff = off + 2 * nv;  // after nv (condition, slots) pairs
    os << " ";
    for (int s = 0; s < NS; ++s) {
      const double a = P[toff + 2 * s], b = P[toff + 2 * s + 1];
      if (x & M_STAB) {
        if (a == 0.0 && b == 0.0) continue;  // identity entry
        os << " pshear(v" << s << ", " << kc.pair(a, b) << ");";
      } else {
        if (a == 1.0 && b == 0.0) continue;
        os << " cscale(v" << s << ", " << kc.pair(a, b) << ");";
      }
    }
    os << "\n";
    // tile-uniform sign terms: branch-free integer flips of the table's output
    for (uint32_t j = 0; j < nv; ++j) {
      const uint64_t gc = raw_bits(P[off + 2 * j]);
      const uint32_t slots = static_cast<uint32_t>(raw_bits(P[off + 2 * j + 1]));
      std::string flips;
      for (int s = 0; s < NS; ++s)
        if ((slots >> s) & 1u) flips += " flip2(v" + std::to_string(s) + ", sg);";
      if (flips.empty()) continue;
      os << "  { const u32 sg = ((g & " << hexu(gc) << ") == " << hexu(gc) << ") ? 0x80000000u : 0u;"
         << flips << " }\n";
    }
    off = toff + 2 * NS;
  }
  if (x & M_SIGN) {
    const uint32_t nt = y >> 16, base = y & 0xffffu;
    if (nt == 0) {
      os << " ";
      for (int s = 0; s < NS; ++s)
        if ((base >> s) & 1u) os << " neg2(v" << s << ");";
      os << "\n";
    } else {
      os << "  { u32 m = " << base << "u;";
      for (uint32_t k = 0; k < nt; ++k) {
        const uint64_t w0 = raw_bits(P[off + 2 * k]), gcond = raw_bits(P[off + 2 * k + 1]);
        const uint32_t slots = static_cast<uint32_t>(w0), lc = static_cast<uint32_t>(w0 >> 32);
        os << " m ^= (";
        if (lc) os << "(jb & " << lc << "u) == " << lc << "u";
        if (lc && gcond) os << " && ";
        if (gcond) os << "(g & " << hexu(gcond) << ") == " << hexu(gcond);
        if (!lc && !gcond) os << "true";
        os << ") ? " << slots << "u : 0u;";
      }
      for (int s = 0; s < NS; ++s) os << " flip2(v" << s << ", (m << " << (31 - s) << ") & 0x80000000u);";
      os << " }\n";
    }
    off += 2 * nt;
  }
  const uint32_t rmask = (x >> M_ROT_SHIFT) & 15u, dmask = (x >> M_DENSE_SHIFT) & 15u;
  for (int a = 0; a < R; ++a) {
    if (!(rmask & (1u << a))) continue;
    const double ck = P[off], form = P[off + 1];
    off += 2;
    os << " ";
    for (int s = 0; s < NS; ++s) {
      if (s & (1 << a)) continue;
      os << (form != 0.0 ? " urot(v" : " trot(v") << s << ", v" << (s | (1 << a)) << ", " << kc(ck) << ");";
    }
    os << "\n";
  }
  for (int a = 0; a < R; ++a) {
    if (!(dmask & (1u << a))) continue;
    std::string m;
    for (int k = 0; k < 8; ++k) m += ", " + kc(P[off + k]);
    off += 8;
    os << " ";
    for (int s = 0; s < NS; ++s) {
      if (s & (1 << a)) continue;
      os << " dense(v" << s << ", v" << (s | (1 << a)) << m << ");";
    }
    os << "\n";
  }
}

// ---- NVRTC (dlopen) --------------------------------------------------------
struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) logsize = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubinsize = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcGetErrorString) errstr = nullptr;
  decltype(&nvrtcVersion) version = nullptr;
  std::string why;
  bool ok = false;
};

const Nvrtc& nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      r.why = "libnvrtc.so.12 not found";
      return r;
    }
#define QT_SYM(f, s)                                           \
  r.f = reinterpret_cast<decltype(r.f)>(dlsym(h, #s));         \
  if (!r.f) {                                                  \
    r.why = "nvrtc symbol " #s " missing";                     \
    return r;                                                  \
  }
    QT_SYM(create, nvrtcCreateProgram)
    QT_SYM(compile, nvrtcCompileProgram)
    QT_SYM(logsize, nvrtcGetProgramLogSize)
    QT_SYM(log, nvrtcGetProgramLog)
    QT_SYM(cubinsize, nvrtcGetCUBINSize)
    QT_SYM(cubin, nvrtcGetCUBIN)
    QT_SYM(destroy, nvrtcDestroyProgram)
    QT_SYM(errstr, nvrtcGetErrorString)
    QT_SYM(version, nvrtcVersion)
#undef QT_SYM
    r.ok = true;
    return r;
  }();
  return n;
}

std::vector<char> compile_cubin_nvrtc(const std::string& src) {
  const Nvrtc& n = nvrtc();
  if (!n.ok) throw std::runtime_error("compiled passes unavailable: " + n.why);
  nvrtcProgram prog;
  if (n.create(&prog, src.c_str(), "qtjit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    throw std::runtime_error("nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "--device-as-default-execution-space"};
  const nvrtcResult rc = n.compile(prog, 3, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t ls = 0;
    n.logsize(prog, &ls);
    std::string log(ls, '\0');
    n.log(prog, &log[0]);
    n.destroy(&prog);
    throw std::runtime_error(std::string("nvrtc: ") + n.errstr(rc) + "\n" + log.substr(0, 2000));
  }
  size_t cs = 0;
  n.cubinsize(prog, &cs);
  std::vector<char> bin(cs);
  n.cubin(prog, bin.data());
  n.destroy(&prog);
  return bin;
}

std::atomic<uint64_t> g_disk_hits{0}, g_disk_writes{0};

// ---- persistent cubin cache -------------------------------------------------
// A fresh process pays no NVRTC for passes some earlier process compiled: the
// CUBIN of every compiled pass is kept on disk under
//   $QTB_JIT_CACHE_DIR  (empty or "off": no disk cache), else
//   $XDG_CACHE_HOME/qtask_b200, else $HOME/.cache/qtask_b200,
// in a file named by a 128-bit hash of (NVRTC version, compile options, the
// generated source). The file stores the source itself and a hit requires it
// to match byte for byte, so neither a hash collision nor a changed code
// generator can return a stale kernel. Files are written to a temporary name
// and renamed (concurrent processes never see partial entries).
constexpr const char* kJitOptions = "sm_100a;c++17;device-default";
constexpr size_t kDiskCacheMaxFiles = 8192;  // no new entries beyond this many

struct DiskCache {
  std::string dir;  // empty: disabled
  std::string tag;  // NVRTC version + options
  std::atomic<size_t> files{0};
};

DiskCache& disk_cache() {
  static DiskCache* dc = [] {
    auto* d = new DiskCache();
    std::string dir;
    if (const char* e = std::getenv("QTB_JIT_CACHE_DIR")) {
      dir = e;
      if (dir.empty() || dir == "off" || dir == "0") return d;
    } else if (const char* x = std::getenv("XDG_CACHE_HOME"); x && *x) {
      dir = std::string(x) + "/qtask_b200";
    } else if (const char* h = std::getenv("HOME"); h && *h) {
      dir = std::string(h) + "/.cache/qtask_b200";
    } else {
      return d;
    }
    // mkdir -p
    for (size_t i = 1; i <= dir.size(); ++i)
      if (i == dir.size() || dir[i] == '/') {
        const std::string part = dir.substr(0, i);
        if (::mkdir(part.c_str(), 0755) != 0 && errno != EEXIST) return d;
      }
    if (::access(dir.c_str(), W_OK | X_OK) != 0) return d;
    size_t n = 0;
    if (DIR* dp = ::opendir(dir.c_str())) {
      while (::readdir(dp)) ++n;
      ::closedir(dp);
    }
    d->files = n;
    int major = 0, minor = 0;
    if (nvrtc().ok) nvrtc().version(&major, &minor);
    d->tag = "nvrtc " + std::to_string(major) + "." + std::to_string(minor) + ";" + kJitOptions;
    d->dir = dir;
    return d;
  }();
  return *dc;
}

uint64_t fnv1a(const std::string& a, const std::string& b, uint64_t h) {
  for (const std::string* s : {&a, &b})
    for (unsigned char c : *s) {
      h ^= c;
      h *= 0x100000001b3ull;
    }
  return h;
}

std::string disk_path(const DiskCache& dc, const std::string& src) {
  char name[40];
  std::snprintf(name, sizeof(name), "%016llx%016llx.qtc",
                static_cast<unsigned long long>(fnv1a(dc.tag, src, 0xcbf29ce484222325ull)),
                static_cast<unsigned long long>(fnv1a(src, dc.tag, 0x9e3779b97f4a7c15ull)));
  return dc.dir + "/" + name;
}

// file: "QTC1" | u64 tag_len | tag | u64 src_len | src | u64 bin_len | bin
bool disk_read(const std::string& path, const std::string& tag, const std::string& src, std::vector<char>* bin) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  bool ok = false;
  char magic[4];
  auto get = [&](std::string* out) {
    uint64_t n = 0;
    if (std::fread(&n, 8, 1, f) != 1 || n > (uint64_t(1) << 30)) return false;
    out->resize(n);
    return n == 0 || std::fread(&(*out)[0], 1, n, f) == n;
  };
  std::string t, s, b;
  if (std::fread(magic, 1, 4, f) == 4 && std::memcmp(magic, "QTC1", 4) == 0 && get(&t) && t == tag && get(&s) &&
      s == src && get(&b) && !b.empty()) {
    bin->assign(b.begin(), b.end());
    ok = true;
  }
  std::fclose(f);
  return ok;
}

void disk_write(DiskCache& dc, const std::string& path, const std::string& src, const std::vector<char>& bin) {
  if (dc.files.load() >= kDiskCacheMaxFiles) return;
  static std::atomic<unsigned> seq{0};
  const std::string tmp = path + ".tmp" + std::to_string(::getpid()) + "_" + std::to_string(seq.fetch_add(1));
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return;
  auto put = [&](const void* p, uint64_t n) { return std::fwrite(&n, 8, 1, f) == 1 && (n == 0 || std::fwrite(p, 1, n, f) == n); };
  const bool ok = std::fwrite("QTC1", 1, 4, f) == 4 && put(dc.tag.data(), dc.tag.size()) && put(src.data(), src.size()) &&
                  put(bin.data(), bin.size());
  if (std::fclose(f) != 0 || !ok || std::rename(tmp.c_str(), path.c_str()) != 0) {
    std::remove(tmp.c_str());
    return;
  }
  dc.files.fetch_add(1);
  g_disk_writes.fetch_add(1);
}

std::vector<char> compile_cubin(const std::string& src) {
  DiskCache& dc = disk_cache();
  if (dc.dir.empty()) return compile_cubin_nvrtc(src);
  const std::string path = disk_path(dc, src);
  std::vector<char> bin;
  if (disk_read(path, dc.tag, src, &bin)) {
    g_disk_hits.fetch_add(1);
    return bin;
  }
  bin = compile_cubin_nvrtc(src);
  disk_write(dc, path, src, bin);
  return bin;
}

struct CacheEntry {
  cudaLibrary_t lib = nullptr;
  JitKernel k;
};

std::mutex& g_mu = *new std::mutex();  // never destroyed (background workers)
std::unordered_map<std::string, CacheEntry>& cache() {
  static auto* m = new std::unordered_map<std::string, CacheEntry>();  // never destroyed
  return *m;
}
JitStats g_stats;

}  // namespace

// What a compiled pass bakes in: the same tile geometry the interpreter
// kernel gets in its KPassHead, plus the rounds.
namespace {

uint32_t swz_map(uint32_t j, const uint8_t* v, int k) {
  uint32_t m = j;
  for (int b = 3; b < k; ++b)
    if ((j >> b) & 1u) m ^= v[b];
  return m;
}

// GF(2) rank of up to three 3-bit vectors
int rank3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t basis[3];
  int n = 0;
  for (uint32_t x : {a, b, c}) {
    for (int i = 0; i < n; ++i) x = std::min(x, x ^ basis[i]);
    if (x) basis[n++] = x;
  }
  return n;
}

// Extra smem wavefronts of a swizzle over the rounds' lane patterns: a
// quarter-warp's 8 lanes differ in the round's three lowest thread (non-
// register) tile bits; they hit 8 distinct bank groups iff those bits'
// contributions are linearly independent.
int swizzle_conflicts(const std::vector<std::array<int, 3>>& lanes, const uint8_t* v) {
  int extra = 0;
  auto contrib = [&](int b) -> uint32_t { return b < 3 ? (1u << b) : v[b]; };
  for (const auto& t : lanes) extra += (8 >> rank3(contrib(t[0]), contrib(t[1]), contrib(t[2]))) - 1;
  return extra;
}

}  // namespace

JitPassSpec make_jit_spec(const PlanPass& ps, int reg_bits, int buf_bits, bool check) {
  JitPassSpec sp;
  const int k = static_cast<int>(ps.tile_phys.size());
  const int R = std::min(reg_bits, k);
  sp.k = k;
  sp.R = R;
  sp.check = check;
  sp.ntiles = 1ull << (buf_bits - k);
  uint64_t tile_mask = 0;
  for (int i = 0; i < k; ++i) {
    const uint64_t b = 1ull << ps.tile_phys[i];
    tile_mask |= b;
    if (i < k - R) sp.lo_mask |= b;
  }
  sp.outer_mask = ((1ull << buf_bits) - 1) & ~tile_mask;
  for (uint32_t s = 0; s < (1u << R); ++s) {
    uint64_t off = 0;
    for (int i = 0; i < R; ++i)
      if ((s >> i) & 1u) off |= 1ull << ps.tile_phys[k - R + i];
    sp.slot_gb[s] = off * sizeof(double2);
  }
  sp.tile_phys = ps.tile_phys;
  // the ring kernel (jit_source_ring): 3 tile buffers must fit one CTA's
  // shared memory and 2 groups one CTA (QTB_JIT_RING=0: the direct kernel)
  static const bool ring_env = [] {
    const char* e = std::getenv("QTB_JIT_RING");
    return !e || std::atoi(e) != 0;
  }();
  sp.ring = ring_env && 3 * (sizeof(double2) << k) + 64 <= 227 * 1024 && (2 << (k - R)) <= 1024 &&
            (1 << (k - R)) >= 32 && buf_bits - k >= 1;
  // measured slower on C3 (247 vs 195 ms: the parameter-bank loads spill
  // registers), so off unless QTB_JIT_KPARAM=1
  static const bool kparam_env = [] {
    const char* e = std::getenv("QTB_JIT_KPARAM");
    return e && std::atoi(e) != 0;
  }();
  sp.kparam = sp.ring && kparam_env;
  // TMA stores need runs of >= 4 amplitudes (64 B) contiguous in the tile
  static const int tma_env = [] {
    const char* e = std::getenv("QTB_JIT_TMA");
    return e ? std::atoi(e) : 0;
  }();
  {
    int run = 0;
    while (run < k && ps.tile_phys[run] == run) ++run;
    sp.tma_store = (sp.ring && run >= 2) ? tma_env : 0;
    if (sp.tma_store == 2 && (k - R < 5 || run < 3)) sp.tma_store = 0;  // whole warps, runs of >= 128 B
    // ... and the per-warp staging areas must fit beside the three tile buffers
    if (sp.tma_store == 2 &&
        3 * (sizeof(double2) << k) + 1024 + (static_cast<size_t>(2) << (k - R)) / 32 * 2048 > 227 * 1024)
      sp.tma_store = 0;
  }
  static const int debug_env = [] {
    const char* e = std::getenv("QTB_JIT_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  sp.debug = debug_env;
  if (sp.debug & (4 | 8 | 16)) sp.check = false;  // timing ablations compute garbage
  if (sp.debug) sp.tma_store = 0;                 // test / ablation builds use the st.global path
  // the smem swizzle: the default (qt_device.cuh swz), or for the ring kernel
  // the first of a fixed pseudo-random sequence of maps that leaves no round
  // with bank conflicts (C5: 71 of 244 rounds conflict under the default)
  for (int b = 3; b < k; ++b) sp.swzv[b] = static_cast<uint8_t>(1u << (b % 3));
  if (sp.ring) {
    std::vector<std::array<int, 3>> lanes;
    for (const PlanRound& pr : ps.rounds) {
      std::array<int, 3> t{};
      int nt = 0;
      for (int b = 0; b < k && nt < 3; ++b)
        if (std::find(pr.reg.begin(), pr.reg.end(), b) == pr.reg.end()) t[nt++] = b;
      if (nt == 3) lanes.push_back(t);
    }
    int best = swizzle_conflicts(lanes, sp.swzv);
    uint32_t rng = 0x9e3779b9u;
    uint8_t cand[kMaxTileBits + 3] = {};
    for (int tries = 0; best > 0 && tries < 4096; ++tries) {
      for (int b = 3; b < k; ++b) {
        rng = rng * 1664525u + 1013904223u;
        cand[b] = static_cast<uint8_t>((rng >> 29) & 7u);
      }
      const int c = swizzle_conflicts(lanes, cand);
      if (c < best) {
        best = c;
        std::copy(cand, cand + k, sp.swzv);
      }
    }
  }
  for (uint32_t s = 0; s < (1u << R); ++s) sp.slot_sb[s] = swz_map(s << (k - R), sp.swzv, k) << 4;
  sp.rounds.resize(ps.rounds.size());
  for (size_t r = 0; r < ps.rounds.size(); ++r) {
    const PlanRound& pr = ps.rounds[r];
    DRound& dr = sp.rounds[r];
    dr = DRound{};
    std::vector<int> sorted(pr.reg.begin(), pr.reg.end());
    std::sort(sorted.begin(), sorted.end());
    for (size_t i = 0; i < pr.reg.size() && i < static_cast<size_t>(kMaxRegBits); ++i) {
      dr.reg[i] = static_cast<uint8_t>(pr.reg[i]);
      dr.sreg[i] = static_cast<uint8_t>(sorted[i]);
      dr.sbit[i] = swz_map(1u << pr.reg[i], sp.swzv, k) << 4;
    }
  }
  return sp;
}

namespace {

// Round r reads (writes) its 2^R amplitudes straight from (to) HBM when its
// register bits avoid the tile's coalescing bits: the thread bits then start
// with the lowest physical bits, so a warp's 16-B accesses cover whole runs.
struct Direct {
  bool ok = false;
  uint64_t tmask = 0;                 // physical bits of the thread (non-register) tile bits
  uint64_t off[1 << kMaxRegBits] = {};  // byte offset of slot s
};

Direct direct_round(const JitPassSpec& sp, const DRound& rd) {
  Direct d;
  const int k = sp.k, R = sp.R;
  if (static_cast<int>(sp.tile_phys.size()) != k || sp.coalesce_bits <= 0) return d;
  for (int i = 1; i < k; ++i)
    if (sp.tile_phys[i] <= sp.tile_phys[i - 1]) return d;  // tile bits ascending
  uint32_t regs = 0;
  for (int i = 0; i < R; ++i) regs |= 1u << rd.reg[i];
  for (int b = 0; b < sp.coalesce_bits; ++b) {
    // physical bit b must be a thread bit of the tile; a shrunk tile's run
    // of low bits may be shorter than coalesce_bits (the bits above the run
    // are outer bits then: nothing to check)
    int ti = -1;
    for (int i = 0; i < k; ++i)
      if (sp.tile_phys[i] == b) ti = i;
    if (ti < 0) {
      if (b == 0) return d;
      break;
    }
    if ((regs >> ti) & 1u) return d;
  }
  for (int i = 0; i < k; ++i)
    if (!((regs >> i) & 1u)) d.tmask |= 1ull << sp.tile_phys[i];
  for (int s = 0; s < (1 << R); ++s) {
    uint64_t o = 0;
    for (int i = 0; i < R; ++i)
      if ((s >> i) & 1) o |= 1ull << sp.tile_phys[rd.reg[i]];
    d.off[s] = o * 16;
  }
  d.ok = true;
  return d;
}

}  // namespace

// Ring variant (the default for compiled passes): a persistent CTA per SM
// with TWO consumer groups of 2^(k-R) threads, each group running the
// register rounds of its own tile, and a ring of three tile buffers in shared
// memory. When a group has finished reading its tile's buffer it streams the
// tile three ahead into that buffer (cp.async 16-B copies, swizzled like every
// round's accesses) and arms the buffer's mbarrier with
// cp.async.mbarrier.arrive; the other group waits on that barrier. So the HBM
// reads of a tile are in flight while both groups compute: no round-0 load
// stalls the FP64 rounds. The last round stores straight to HBM when its
// register bits leave the coalescing bits to the threads.
//   tile j (of the CTA's range) -> group j & 1, buffer j % 3, mbarrier j % 6
//   with phase parity (j / 6) & 1. Six barriers, not three: tiles j and j + 3
// share a buffer but belong to different groups, and the group waiting for
// j + 3 may get there while the load of tile j is still in flight -- with one
// barrier per buffer its parity test would then see tile j's pending phase as
// the "preceding" phase of j + 3's and pass. Barrier j % 6 was last used by
// tile j - 6 of the same group, which that group has consumed.
std::string jit_source_ring(const JitPassSpec& sp, const MicroPass& mp, std::vector<double>* kparams) {
  const int R = sp.R, NS = 1 << R, k = sp.k;
  const int T = 1 << (k - R);
  const size_t nr = sp.rounds.size();
  const uint32_t TB = 16u << k;
  std::ostringstream os;
  Consts kc;
  kc.param = sp.kparam;
  const Direct dl = nr ? direct_round(sp, sp.rounds.back()) : Direct{};
  // QTB_JIT_DEBUG (test builds): bit 0 -- every shared / global index is
  // range-checked (a violation sets flag bit 2 and skips the access: the
  // state's sync raises); bit 1 -- the two groups are skewed by pseudo-
  // random sleeps, so the mbarrier / named-barrier protocol meets other
  // interleavings (the results must not change by a bit)
  const bool bounds = (sp.debug & 1) != 0, skew = (sp.debug & 2) != 0;
  // timing ablations (WRONG results, profiling only): 4 -- the HBM stores are
  // skipped (behind a run-time-false test, so the arithmetic stays), 8 -- the
  // cp.async tile loads likewise, 16 -- no arithmetic
  const bool no_st = (sp.debug & 4) != 0, no_ld = (sp.debug & 8) != 0, no_fp = (sp.debug & 16) != 0;
  const std::string st_guard = no_st ? "if (per == 0xffffffffffffull) " : "";
  const uint64_t amps = sp.ntiles << k;
  auto ok_s = [&](const std::string& off) {  // shared byte offset within a tile buffer
    return bounds ? "if ((" + off + ") >= " + std::to_string(TB) + "u) { atomicOr(flag, 4); } else " : std::string();
  };
  const std::string outer = hexu(sp.outer_mask);
  // element offsets fit 32 bits for buffers of <= 2^32 amplitudes
  const bool narrow = sp.ntiles <= (1ull << 20) && (sp.lo_mask >> 32) == 0 && (sp.outer_mask >> 32) == 0 &&
                      (dl.tmask >> 32) == 0;
  const char* ix = narrow ? "u32" : "u64";
  // TMA store geometry: the tile's lowest c bits are physical bits 0..c-1, so
  // its amplitudes form 2^(k-c) runs of 2^c contiguous amplitudes; run r sits
  // at shared byte r * run_bytes of the (unswizzled) staging layout. Thread t
  // issues runs t, t + T, ... (rpt of them), or the first nruns threads one.
  const bool tma = sp.tma_store == 1;
  const bool wdrain = sp.tma_store == 2;
  const uint32_t stage_off = 3 * TB + 1024;  // per-warp staging areas (wdrain), after the mbarriers
  int crun = 0;
  while (crun < k && sp.tile_phys[crun] == crun) ++crun;
  const uint32_t run_bytes = 16u << crun;
  const uint32_t nruns = 1u << (k - crun);
  const uint32_t rpt = nruns > static_cast<uint32_t>(T) ? nruns / T : 1u;
  const uint32_t run_threads = std::min<uint32_t>(nruns, T);
  uint64_t run_tmask = 0;              // physical bits the issuing thread's index deposits into
  std::vector<uint64_t> run_off(rpt, 0);  // amplitude offset of the thread's i-th run
  {
    int tb = 0;
    while ((1u << tb) < run_threads) ++tb;
    for (int b = 0; b < tb; ++b) run_tmask |= 1ull << sp.tile_phys[crun + b];
    for (uint32_t i = 0; i < rpt; ++i)
      for (int b = 0; crun + tb + b < k; ++b)
        if ((i >> b) & 1u) run_off[i] |= 1ull << sp.tile_phys[crun + tb + b];
  }
  static const bool asm_smem = [] {
    const char* e = std::getenv("QTB_JIT_ASMSMEM");
    return e && std::atoi(e) != 0;
  }();
  // Fused exchange: destination of the amplitude at local index x (its thread
  // part xt = tile base + thread offset at run time, its slot part a literal):
  //   rank   = peer[v],  v bit i = bit fuse_v[i] of x
  //   index  = (x with the victim bits cleared) | rfix
  // emit_fused_ptrs declares one base pointer per pattern of the victim bits
  // that sit in the slot offsets (literal per slot); fused_ptr(s) names the
  // pointer of slot s and fused_off(s) its literal byte offset.
  const bool fuse = sp.fuse_k > 0;
  uint64_t fuse_vmask = 0;
  for (int i = 0; i < sp.fuse_k; ++i) fuse_vmask |= 1ull << sp.fuse_v[i];
  auto fuse_pattern = [&](uint64_t off_bytes) {  // victim bits spelled by a slot's byte offset
    uint32_t v = 0;
    for (int i = 0; i < sp.fuse_k; ++i)
      if ((off_bytes / 16) >> sp.fuse_v[i] & 1ull) v |= 1u << i;
    return v;
  };
  auto emit_fused_ptrs = [&](const std::string& xt, const uint64_t* off) {
    uint64_t slot_bits = 0;
    for (int s2 = 0; s2 < NS; ++s2) slot_bits |= off[s2] / 16;
    os << "      u32 vr = 0;\n";
    for (int i = 0; i < sp.fuse_k; ++i)
      if (!((slot_bits >> sp.fuse_v[i]) & 1ull))
        os << "      vr |= static_cast<u32>((u64(" << xt << ") >> " << sp.fuse_v[i] << ") & 1ull) << " << i << ";\n";
    os << "      const u64 xk = (u64(" << xt << ") & ~" << hexu(fuse_vmask) << ") | fx.rfix;\n";
    std::vector<char> seen(8, 0);
    for (int s2 = 0; s2 < NS; ++s2) {
      const uint32_t q = fuse_pattern(off[s2]);
      if (seen[q]) continue;
      seen[q] = 1;
      os << "      char* const fp" << q << " = reinterpret_cast<char*>(fx.peer[vr | " << q << "u] + xk);\n";
    }
  };
  auto fused_ptr = [&](uint64_t off_bytes) { return "fp" + std::to_string(fuse_pattern(off_bytes)); };
  auto fused_off = [&](uint64_t off_bytes) { return off_bytes & ~(fuse_vmask * 16); };
  static const bool early = [] {
    const char* e = std::getenv("QTB_JIT_EARLY");
    return !e || std::atoi(e) != 0;
  }();
  // this pass's smem swizzle (make_jit_spec: no bank conflicts in any round)
  os << "FI u32 swzp(u32 j) {\n  u32 m = j;\n";
  for (int bb = 3; bb < k; ++bb)
    if (sp.swzv[bb]) os << "  m ^= (0u - ((j >> " << bb << ") & 1u)) & " << int(sp.swzv[bb]) << "u;\n";
  os << "  return m;\n}\n";
  os << "FI void mbar_wait(u32 a, u32 ph) {\n"
     << "  asm volatile(\"{\\n .reg .pred p;\\n W:\\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\\n"
        " @!p bra W;\\n }\" :: \"r\"(a), \"r\"(ph) : \"memory\");\n}\n"
     << "FI void gbar(u32 id) { asm volatile(\"bar.sync %0, " << T << ";\" :: \"r\"(id) : \"memory\"); }\n"
     // smaller tiles: several CTAs per SM (512 threads of <= 128 registers in all)
     << "extern \"C\" __global__ void __launch_bounds__(" << 2 * T << ", " << std::max(1, 512 / (2 * T)) << ")\n"
     << "qtjit(double2* psi, const double2* src, int* flag, u64 gbase_hi, u64 per"
     << (sp.kparam ? ", const __grid_constant__ KP K" : "")
     << (fuse ? ", const __grid_constant__ FX fx" : "") << ") {\n"
     << "  extern __shared__ __align__(16) double2 sm[];\n"
     << "  char* const sm0 = reinterpret_cast<char*>(sm);\n"
     << "  const u32 smbase = static_cast<u32>(__cvta_generic_to_shared(sm0));\n"
     << "  const u32 fb = smbase + " << 3 * TB << "u;  // 6 mbarriers (8 B each)\n"
     << "  const u32 grp = threadIdx.x >> " << (k - R) << ";\n"
     << "  const u32 t = threadIdx.x & " << (T - 1) << "u;\n"
     << "  const " << ix << " off_t = pdep64(t, " << hexu(sp.lo_mask) << ");\n"
     << "  const u32 st4 = swzp(t) << 4;\n";
  if (dl.ok && !tma) os << "  const " << ix << " off_dl = pdep64(t, " << hexu(dl.tmask) << ");\n";
  if (tma) os << "  const u64 off_run = pdep64(t, " << hexu(run_tmask) << ");\n";
  // tile counters in 32 bits (<= 2^28 tiles): fewer live registers
  os << "  const u32 t0 = blockIdx.x * static_cast<u32>(per);\n"
     << "  const u32 t1 = t0 + static_cast<u32>(per) < " << sp.ntiles << "u ? t0 + static_cast<u32>(per) : "
     << sp.ntiles << "u;\n"
     << "  const u32 cnt = t1 > t0 ? t1 - t0 : 0u;\n"
     << "  if (threadIdx.x == 0) {\n"
     << "    for (u32 b = 0; b < 6; ++b)\n"
     << "      asm volatile(\"mbarrier.init.shared::cta.b64 [%0], %1;\" :: \"r\"(fb + 8 * b), \"r\"(" << T
     << ") : \"memory\");\n"
     << "  }\n"
     << "  __syncthreads();\n"
     << "  auto load = [&](u32 i) {\n"
     << "    const char* s = reinterpret_cast<const char*>(src + static_cast<" << ix << ">(pdep64(t0 + i, " << outer
     << ")) + off_t);\n"
     << "    const u32 b = static_cast<u32>(i % 3);\n"
     << "    const u32 d = smbase + b * " << TB << "u;\n";
  // the swizzled smem address is formed inside each asm statement: as
  // plain C++ the 2^R loop-invariant (st4 ^ slot) values would be hoisted
  // out of the tile loop and pin 2^R registers (spills at 128)
  if (bounds)
    os << "    if (u64(pdep64(t0 + i, " << outer << ")) + off_t + " << (sp.slot_gb[NS - 1] / 16) << "ull >= " << amps
       << "ull || (st4 ^ " << sp.slot_sb[NS - 1] << "u) >= " << TB << "u) atomicOr(flag, 4);\n";
  if (no_ld) os << "    if (per == 0xffffffffffffull) {\n";
  for (int s2 = 0; s2 < NS; ++s2)
    os << "    asm volatile(\"{ .reg .b32 q; xor.b32 q, %0, " << sp.slot_sb[s2]
       << "; add.u32 q, q, %1; cp.async.cg.shared.global [q], [%2], 16; }\" :: \"r\"(st4), \"r\"(d), \"l\"(s + "
       << sp.slot_gb[s2] << "ull) : \"memory\");\n";
  if (no_ld) os << "    }\n";
  os << "    asm volatile(\"cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\" :: \"r\"(fb + 8 * static_cast<u32>(i % 6)) : \"memory\");\n"
     << "  };\n"
     << "  if (grp == 0) { if (cnt > 0) load(0); if (cnt > 2) load(2); }\n"
     << "  else if (cnt > 1) load(1);\n"
     << "  bool bad = false;\n";
  os << "  for (u32 j = grp; j < cnt; j += 2) {\n"
     << "    const u32 bi = static_cast<u32>(j % 3);\n"
     << "    const u32 smb = smbase + bi * " << TB << "u;\n"
     << "    char* const smp = sm0 + bi * " << TB << "u;\n"
     << "    mbar_wait(fb + 8 * static_cast<u32>(j % 6), static_cast<u32>((j / 6) & 1));\n"
     << "    const " << ix << " base = static_cast<" << ix << ">(pdep64(t0 + j, " << outer << "));\n"
     << "    const u64 g = gbase_hi | base;\n";
  if (skew)
    os << "    if (((j * 2654435761u) >> 29) == grp) __nanosleep(((j * 40503u) & 1023u) + 64u);\n";
  // ---- TMA-store variant of the tile body -------------------------------
  // The buffer of this group's previous tile (j - 2) is being read by its
  // bulk stores; it is refilled with tile j + 1 at this tile's first group
  // barrier, after every thread has waited for its own bulk reads.
  auto pin = [&](const char* v) {
    os << "     ";
    for (int s2 = 0; s2 < NS; ++s2)
      os << " asm volatile(\"\" : \"+d\"(" << v << s2 << ".x), \"+d\"(" << v << s2 << ".y));";
    os << "\n";
  };
  auto first_barrier = [&]() {
    os << "      asm volatile(\"cp.async.bulk.wait_group.read 0;\" ::: \"memory\");\n"
       << "      gbar(1 + grp);\n"
       << "      if (j >= 2 && j + 1 < cnt) load(j + 1);\n";
  };
  auto bulk_stores = [&]() {
    // the staged tile is complete and visible to the async proxy: one bulk
    // copy per run, issued by the threads that own runs
    os << "      asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
       << "      gbar(1 + grp);\n";
    if (run_threads < static_cast<uint32_t>(T)) os << "      if (t < " << run_threads << "u)";
    os << "      {\n        const char* gd = reinterpret_cast<const char*>(psi + base + off_run);\n"
       << "        const u32 ss = smb + t * " << run_bytes << "u;\n";
    for (uint32_t i = 0; i < rpt; ++i)
      os << "        asm volatile(\"cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], " << run_bytes
         << ";\" :: \"l\"(gd + " << run_off[i] * 16 << "ull), \"r\"(ss + " << i * T * run_bytes
         << "u) : \"memory\");\n";
    os << "        asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n      }\n";
  };
  for (size_t r = 0; tma && r < nr; ++r) {
    const DRound& rd = sp.rounds[r];
    const bool last_direct = r + 1 == nr && dl.ok;
    os << "    { // round " << r << "\n      u32 jb = t;";
    for (int i = 0; i < R; ++i) os << " jb = insert_zero(jb, " << int(rd.sreg[i]) << "u);";
    os << "\n      const u32 a = swzp(jb) << 4;\n     ";
    std::vector<uint32_t> sb(NS, 0), lit(NS, 0);
    for (int s2 = 0; s2 < NS; ++s2)
      for (int i = 0; i < R; ++i)
        if (s2 & (1 << i)) {
          sb[s2] ^= rd.sbit[i];
          lit[s2] |= 16u << rd.reg[i];
        }
    for (int s2 = 0; s2 < NS; ++s2)
      os << " double2 v" << s2 << " = *reinterpret_cast<const double2*>(smp + (a ^ " << sb[s2] << "u));";
    os << "\n";
    const uint32_t w0 = mp.round_first[r], w1 = w0 + mp.round_count[r];
    if (last_direct) {
      // every thread has read the (swizzled) buffer before anyone overwrites
      // it with the unswizzled staging layout
      pin("v");
      if (r == 0) first_barrier();
      else os << "      gbar(1 + grp);\n";
    }
    for (uint32_t w = w0; w < w1; ++w) emit_word(os, kc, R, mp.words[2 * w], mp.words[2 * w + 1], mp.pool);
    os << "     ";
    for (int s2 = 0; s2 < NS; ++s2) {
      if (last_direct) {
        if (sp.check) os << " bad = bad || !finite2(v" << s2 << ");";
        os << " *reinterpret_cast<double2*>(smp + ((jb << 4) | " << lit[s2] << "u)) = v" << s2 << ";";
      } else {
        os << " *reinterpret_cast<double2*>(smp + (a ^ " << sb[s2] << "u)) = v" << s2 << ";";
      }
    }
    os << "\n";
    if (last_direct) {
      bulk_stores();
    } else if (r == 0) {
      first_barrier();
    } else {
      os << "      gbar(1 + grp);\n";
    }
    os << "    }\n";
  }
  if (tma && !dl.ok) {
    // the last round kept low bits in registers: re-read the tile with the
    // coalesced (load) mapping and stage it unswizzled
    os << "    {\n";
    for (int s2 = 0; s2 < NS; ++s2)
      os << "      double2 x" << s2 << " = *reinterpret_cast<const double2*>(smp + (st4 ^ " << sp.slot_sb[s2] << "u));\n";
    pin("x");
    os << "      gbar(1 + grp);\n     ";
    for (int s2 = 0; s2 < NS; ++s2) {
      if (sp.check) os << " bad = bad || !finite2(x" << s2 << ");";
      os << " *reinterpret_cast<double2*>(smp + ((t << 4) | " << (static_cast<uint32_t>(s2) << (k - R + 4)) << "u)) = x" << s2 << ";";
    }
    os << "\n";
    bulk_stores();
    os << "    }\n";
  }
  if (tma && nr == 0) throw std::logic_error("compiled pass without rounds");
  // Warp-staged drain (tma_store == 2): the warp's 2^R result slots leave in
  // batches of two through its own staging area; the lanes that start a
  // contiguous run of 2^cl amplitudes issue one bulk copy per slot. The warp
  // waits for its own bulk reads only (cp.async.bulk.wait_group.read), so a
  // slow drain (HBM write back-pressure) blocks neither the LSU nor the other
  // group's shared-memory traffic.
  auto staged_drain = [&](const char* v, const std::string& gptr, const uint64_t* off, int cl) {
    const uint32_t rb = 16u << cl;
    os << "      {\n        const u32 lane = threadIdx.x & 31u;\n"
       << "        const u32 wst = " << stage_off << "u + (threadIdx.x >> 5) * 2048u + lane * 16u;\n"
       << "        const bool lead = (lane & " << ((1u << cl) - 1) << "u) == 0;\n";
    for (int q = 0; q < NS / 2; ++q) {
      const uint32_t hb = (q & 1) * 1024u;
      os << "        asm volatile(\"cp.async.bulk.wait_group.read 1;\" ::: \"memory\");\n        __syncwarp();\n       ";
      for (int i = 0; i < 2; ++i) {
        const int s2 = 2 * q + i;
        if (sp.check) os << " bad = bad || !finite2(" << v << s2 << ");";
        os << " *reinterpret_cast<double2*>(sm0 + wst + " << (hb + i * 512u) << "u) = " << v << s2 << ";";
      }
      os << "\n        asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n        __syncwarp();\n"
         << "        if (lead) {\n";
      for (int i = 0; i < 2; ++i) {
        const int s2 = 2 * q + i;
        os << "          asm volatile(\"cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], " << rb
           << ";\" :: \"l\"(" << gptr << " + " << off[s2] << "ull), \"r\"(smbase + wst + " << (hb + i * 512u)
           << "u) : \"memory\");\n";
      }
      os << "          asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n        }\n";
    }
    os << "      }\n";
  };
  // lane-contiguous low bits of the last round's direct mapping / of the load mapping
  int cl_direct = 0, cl_load = 0;
  if (wdrain && nr) {
    uint32_t regs = 0;
    for (int i = 0; i < R; ++i) regs |= 1u << sp.rounds.back().reg[i];
    while (cl_direct < 5 && cl_direct < crun && !((regs >> cl_direct) & 1u)) ++cl_direct;
    cl_load = std::min(5, std::min(crun, k - R));
  }
  for (size_t r = 0; !tma && r < nr; ++r) {
    const DRound& rd = sp.rounds[r];
    const bool last_direct = r + 1 == nr && dl.ok;
    os << "    { // round " << r << "\n      u32 jb = t;";
    for (int i = 0; i < R; ++i) os << " jb = insert_zero(jb, " << int(rd.sreg[i]) << "u);";
    os << "\n      const u32 a = swzp(jb) << 4;\n     ";
    std::vector<uint32_t> sb(NS, 0);
    for (int s2 = 0; s2 < NS; ++s2)
      for (int i = 0; i < R; ++i)
        if (s2 & (1 << i)) sb[s2] ^= rd.sbit[i];
    for (int s2 = 0; s2 < NS; ++s2) {
      if (asm_smem)
        os << " double2 v" << s2 << "; asm volatile(\"{ .reg .b32 q; xor.b32 q, %2, " << sb[s2]
           << "; add.u32 q, q, %3; ld.shared.v2.f64 {%0, %1}, [q]; }\" : \"=d\"(v" << s2 << ".x), \"=d\"(v" << s2
           << ".y) : \"r\"(a), \"r\"(smb));";
      else
        os << " double2 v" << s2 << " = make_double2(0.0, 0.0); " << ok_s("a ^ " + std::to_string(sb[s2]) + "u")
           << "v" << s2 << " = *reinterpret_cast<const double2*>(smp + (a ^ " << sb[s2] << "u));";
    }
    os << "\n";
    const uint32_t w0 = mp.round_first[r], w1 = w0 + mp.round_count[r];
    // the group's buffer is free once every thread has read it for the last
    // time: with `early` the refill (tile j + 3) is issued right after the
    // last round's shared-memory reads have landed in registers, before that
    // round's arithmetic, so the HBM read gets the round's compute time as
    // extra lead (the empty asm statements pin the loads before the barrier)
    const bool early_refill = last_direct && early;
    if (early_refill) {
      os << "     ";
      for (int s2 = 0; s2 < NS; ++s2)
        os << " asm volatile(\"\" : \"+d\"(v" << s2 << ".x), \"+d\"(v" << s2 << ".y));";
      os << "\n      gbar(1 + grp);\n"
         << "      if (j + 3 < cnt) load(j + 3);\n";
    }
    for (uint32_t w = w0; w < w1 && !no_fp; ++w) emit_word(os, kc, R, mp.words[2 * w], mp.words[2 * w + 1], mp.pool);
    if (last_direct) {
      if (!early_refill)
        os << "      gbar(1 + grp);\n"
           << "      if (j + 3 < cnt) load(j + 3);\n";
      if (fuse) {
        os << "      {\n";
        emit_fused_ptrs("base + off_dl", dl.off);
        os << "     ";
        for (int s2 = 0; s2 < NS; ++s2) {
          if (sp.check) os << " bad = bad || !finite2(v" << s2 << ");";
          os << " __stcs(reinterpret_cast<double2*>(" << fused_ptr(dl.off[s2]) << " + " << fused_off(dl.off[s2])
             << "ull), v" << s2 << ");";
        }
        os << "\n      }\n    }\n";
        continue;
      }
      os << "      { char* gd = reinterpret_cast<char*>(psi + base + off_dl);\n     ";
      if (wdrain && cl_direct >= 3) {
        os << "\n";
        staged_drain("v", "gd", dl.off, cl_direct);
        os << "      }\n    }\n";
        continue;
      }
      for (int s2 = 0; s2 < NS; ++s2) {
        if (sp.check) os << " bad = bad || !finite2(v" << s2 << ");";
        if (bounds)
          os << " if (u64(base) + off_dl + " << dl.off[s2] / 16 << "ull >= " << amps
             << "ull) atomicOr(flag, 4); else";
        os << " " << st_guard << "__stcs(reinterpret_cast<double2*>(gd + " << dl.off[s2] << "ull), v" << s2 << ");";
      }
      os << " }\n    }\n";
    } else {
      os << "     ";
      for (int s2 = 0; s2 < NS; ++s2) {
        if (asm_smem)
          os << " asm volatile(\"{ .reg .b32 q; xor.b32 q, %0, " << sb[s2]
             << "; add.u32 q, q, %1; st.shared.v2.f64 [q], {%2, %3}; }\" :: \"r\"(a), \"r\"(smb), \"d\"(v" << s2
             << ".x), \"d\"(v" << s2 << ".y) : \"memory\");";
        else
          os << " " << ok_s("a ^ " + std::to_string(sb[s2]) + "u") << "*reinterpret_cast<double2*>(smp + (a ^ "
             << sb[s2] << "u)) = v" << s2 << ";";
      }
      os << "\n      gbar(1 + grp);\n    }\n";
    }
  }
  if (tma) {
    // handled above
  } else if (!dl.ok && (early || fuse)) {
    // copy-out: the whole tile share goes to registers first, so the refill
    // of this buffer starts before the HBM stores are issued
    os << "    {\n      char* d = reinterpret_cast<char*>(psi + base + off_t);\n";
    for (int s2 = 0; s2 < NS; ++s2)
      os << "      double2 x" << s2 << "; asm volatile(\"{ .reg .b32 q; xor.b32 q, %2, " << sp.slot_sb[s2]
         << "; add.u32 q, q, %3; ld.shared.v2.f64 {%0, %1}, [q]; }\" : \"=d\"(x" << s2 << ".x), \"=d\"(x" << s2
         << ".y) : \"r\"(st4), \"r\"(smb));\n";
    os << "     ";
    for (int s2 = 0; s2 < NS; ++s2)
      os << " asm volatile(\"\" : \"+d\"(x" << s2 << ".x), \"+d\"(x" << s2 << ".y));";
    os << "\n      gbar(1 + grp);\n"
       << "      if (j + 3 < cnt) load(j + 3);\n";
    if (fuse) {
      emit_fused_ptrs("base + off_t", sp.slot_gb);
      for (int s2 = 0; s2 < NS; ++s2) {
        os << "     ";
        if (sp.check) os << " bad = bad || !finite2(x" << s2 << ");";
        os << " __stcs(reinterpret_cast<double2*>(" << fused_ptr(sp.slot_gb[s2]) << " + " << fused_off(sp.slot_gb[s2])
           << "ull), x" << s2 << ");\n";
      }
    } else if (wdrain && cl_load >= 3) {
      staged_drain("x", "d", sp.slot_gb, cl_load);
    }
    for (int s2 = 0; s2 < NS && !fuse && !(wdrain && cl_load >= 3); ++s2) {
      os << "     ";
      if (sp.check) os << " bad = bad || !finite2(x" << s2 << ");";
      os << " " << st_guard << "__stcs(reinterpret_cast<double2*>(d + " << sp.slot_gb[s2] << "ull), x" << s2 << ");\n";
    }
    os << "    }\n";
  } else if (!dl.ok) {
    os << "    {\n      char* d = reinterpret_cast<char*>(psi + base + off_t);\n";
    for (int s2 = 0; s2 < NS; ++s2) {
      os << "      { double2 x; asm volatile(\"{ .reg .b32 q; xor.b32 q, %2, " << sp.slot_sb[s2]
         << "; add.u32 q, q, %3; ld.shared.v2.f64 {%0, %1}, [q]; }\" : \"=d\"(x.x), \"=d\"(x.y) : \"r\"(st4), \"r\"(smb));";
      if (sp.check) os << " bad = bad || !finite2(x);";
      os << " __stcs(reinterpret_cast<double2*>(d + " << sp.slot_gb[s2] << "ull), x); }\n";
    }
    os << "    }\n"
       << "    gbar(1 + grp);\n"
       << "    if (j + 3 < cnt) load(j + 3);\n";
  }
  os << "  }\n";
  if (tma || wdrain) os << "  asm volatile(\"cp.async.bulk.wait_group 0;\" ::: \"memory\");\n";
  if (sp.check) os << "  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);\n";
  os << "}\n";
  std::string head = kPrelude;
  if (fuse) head += "struct FX { double2* peer[8]; u64 rfix; };\n";
  if (sp.kparam) {
    if (kc.vals.size() > kMaxKParams) {
      // too many constants for one parameter block: literals instead
      JitPassSpec lit = sp;
      lit.kparam = false;
      if (kparams) kparams->clear();
      return jit_source_ring(lit, mp, kparams);
    }
    if (kc.vals.empty()) kc.vals.push_back(0.0);
    head += "struct KP { double k[" + std::to_string(kc.vals.size()) + "]; };\n";
    if (kparams) *kparams = kc.vals;
  }
  return head + os.str();
}

std::string jit_source(const JitPassSpec& sp, const MicroPass& mp, std::vector<double>* kparams) {
  const int R = sp.R, NS = 1 << R, k = sp.k;
  if (sp.ring) return jit_source_ring(sp, mp, kparams);
  const int threads = 1 << (k - R);
  const size_t nr = sp.rounds.size();
  std::ostringstream os;
  Consts kc;
  // first / last round straight from / to HBM (no staging through smem)
  const Direct d0 = (!sp.pipe && nr) ? direct_round(sp, sp.rounds.front()) : Direct{};
  const Direct dl = nr ? direct_round(sp, sp.rounds.back()) : Direct{};
  // launch bounds: <= 64 registers for R <= 3, <= 128 for R = 4
  const int minb = sp.min_blocks > 0 ? sp.min_blocks : std::max(1, (R >= 4 ? 512 : 1024) / threads);
  os << "extern \"C\" __global__ void __launch_bounds__(" << threads << ", " << minb << ")\n"
     << "qtjit(double2* psi, const double2* src, int* flag, u64 gbase_hi, u64 per) {\n"
     << "  extern __shared__ double2 sm[];\n"
     << (sp.pipe ? "" : "  char* const smb = reinterpret_cast<char*>(sm);\n")
     << "  const u32 t = threadIdx.x;\n"
     << "  const u64 off_t = pdep64(t, " << hexu(sp.lo_mask) << ");\n"
     << "  const u32 st4 = swz(t) << 4;\n";
  if (d0.ok) os << "  const u64 off_d0 = pdep64(t, " << hexu(d0.tmask) << ");\n";
  if (dl.ok) os << "  const u64 off_dl = pdep64(t, " << hexu(dl.tmask) << ");\n";
  os << "  const u64 t0 = u64(blockIdx.x) * per;\n"
     << "  const u64 t1 = t0 + per < " << hexu(sp.ntiles) << " ? t0 + per : " << hexu(sp.ntiles) << ";\n"
     << "  u64 base = pdep64(t0, " << hexu(sp.outer_mask) << ");\n"
     << "  bool bad = false;\n";
  const std::string outer = hexu(sp.outer_mask);
  const uint32_t tbytes = 16u << k;
  auto cp_tile = [&](const std::string& basev, const std::string& dst) {
    os << "      { const char* s = reinterpret_cast<const char*>(src + " << basev << " + off_t);\n"
       << "        const u32 d0 = static_cast<u32>(__cvta_generic_to_shared(" << dst << "));\n";
    for (int s = 0; s < NS; ++s)
      os << "        asm volatile(\"cp.async.cg.shared.global [%0], [%1], 16;\" :: \"r\"(d0 + (st4 ^ "
         << sp.slot_sb[s] << "u)), \"l\"(s + " << sp.slot_gb[s] << "ull) : \"memory\");\n";
    os << "        asm volatile(\"cp.async.commit_group;\" ::: \"memory\"); }\n";
  };
  if (sp.pipe) {
    os << "  char* const sm0 = reinterpret_cast<char*>(sm);\n"
       << "  u32 cur = 0;\n"
       << "  if (t0 < t1) {\n";
    cp_tile("base", "sm0");
    os << "  }\n";
  }
  os << "  for (u64 tile = t0; tile < t1; ++tile) {\n";
  if (sp.pipe) {
    os << "    char* const smb = sm0 + cur;\n"
       << "    if (tile + 1 < t1) {\n"
       << "      const u64 nb = ((base | ~" << outer << ") + 1) & " << outer << ";\n";
    cp_tile("nb", "sm0 + (cur ^ " + std::to_string(tbytes) + "u)");
    os << "      asm volatile(\"cp.async.wait_group 1;\" ::: \"memory\");\n"
       << "    } else {\n"
       << "      asm volatile(\"cp.async.wait_group 0;\" ::: \"memory\");\n"
       << "    }\n"
       << "    __syncthreads();\n";
  } else if (!d0.ok) {
    os << "    {\n      const char* s = reinterpret_cast<const char*>(src + base + off_t);\n";
    for (int s = 0; s < NS; ++s)
      os << "      const double2 l" << s << " = __ldcs(reinterpret_cast<const double2*>(s + "
         << sp.slot_gb[s] << "ull));\n";
    if (sp.pf_bits > 0) {
      const uint32_t run = 1u << sp.pf_bits;
      os << "      if ((t & " << (run - 1) << "u) == 0 && tile + 1 < t1) {\n"
         << "        const char* n = reinterpret_cast<const char*>(src + (((base | ~" << outer << ") + 1) & "
         << outer << ") + off_t);\n";
      for (int s = 0; s < NS; ++s)
        os << "        asm volatile(\"cp.async.bulk.prefetch.L2.global [%0], %1;\" :: \"l\"(n + "
           << sp.slot_gb[s] << "ull), \"r\"(" << (16u * run) << "u) : \"memory\");\n";
      os << "      }\n";
    }
    for (int s = 0; s < NS; ++s)
      os << "      *reinterpret_cast<double2*>(smb + (st4 ^ " << sp.slot_sb[s] << "u)) = l" << s << ";\n";
    os << "    }\n    __syncthreads();\n";
  }
  os << "    const u64 g = gbase_hi | base;\n";
  for (size_t r = 0; r < nr; ++r) {
    const DRound& rd = sp.rounds[r];
    const bool first_direct = r == 0 && d0.ok, last_direct = r + 1 == nr && dl.ok;
    os << "    { // round " << r << "\n      u32 jb = t;";
    for (int i = 0; i < R; ++i) os << " jb = insert_zero(jb, " << int(rd.sreg[i]) << "u);";
    os << "\n      const u32 a = swz(jb) << 4;\n     ";
    std::vector<uint32_t> sb(NS, 0);
    for (int s = 0; s < NS; ++s)
      for (int i = 0; i < R; ++i)
        if (s & (1 << i)) sb[s] ^= rd.sbit[i];
    if (first_direct) {
      os << " const char* gs = reinterpret_cast<const char*>(src + base + off_d0);\n     ";
      for (int s = 0; s < NS; ++s)
        os << " double2 v" << s << " = __ldcs(reinterpret_cast<const double2*>(gs + " << d0.off[s] << "ull));";
      if (sp.pf_bits > 0) {
        // L2 prefetch of the next tile's round-0 data while this tile computes:
        // the threads whose low run bits are zero cover one run per slot
        int run = 0;
        while (run < 12 && ((d0.tmask >> run) & 1ull)) ++run;
        run = std::min(run, sp.pf_bits);
        os << "\n      if ((t & " << ((1u << run) - 1) << "u) == 0 && tile + 1 < t1) {\n"
           << "        const char* n = reinterpret_cast<const char*>(src + (((base | ~" << outer << ") + 1) & "
           << outer << ") + off_d0);\n";
        for (int s = 0; s < NS; ++s)
          os << "        asm volatile(\"cp.async.bulk.prefetch.L2.global [%0], %1;\" :: \"l\"(n + "
             << d0.off[s] << "ull), \"r\"(" << (16u << run) << "u) : \"memory\");\n";
        os << "      }\n     ";
      }
    } else {
      for (int s = 0; s < NS; ++s)
        os << " double2 v" << s << " = *reinterpret_cast<const double2*>(smb + (a ^ " << sb[s] << "u));";
    }
    os << "\n";
    const uint32_t w0 = mp.round_first[r], w1 = w0 + mp.round_count[r];
    for (uint32_t w = w0; w < w1; ++w) emit_word(os, kc, R, mp.words[2 * w], mp.words[2 * w + 1], mp.pool);
    if (last_direct) {
      os << "      { char* gd = reinterpret_cast<char*>(psi + base + off_dl);\n     ";
      for (int s = 0; s < NS; ++s) {
        if (sp.check) os << " bad = bad || !finite2(v" << s << ");";
        os << " __stcs(reinterpret_cast<double2*>(gd + " << dl.off[s] << "ull), v" << s << ");";
      }
      os << " }\n    }\n";
    } else {
      os << "     ";
      for (int s = 0; s < NS; ++s)
        os << " *reinterpret_cast<double2*>(smb + (a ^ " << sb[s] << "u)) = v" << s << ";";
      os << "\n      __syncthreads();\n    }\n";
    }
  }
  if (!dl.ok) {
    os << "    {\n      char* d = reinterpret_cast<char*>(psi + base + off_t);\n";
    for (int s = 0; s < NS; ++s) {
      os << "      { const double2 x = *reinterpret_cast<const double2*>(smb + (st4 ^ " << sp.slot_sb[s]
         << "u));";
      if (sp.check) os << " bad = bad || !finite2(x);";
      os << " __stcs(reinterpret_cast<double2*>(d + " << sp.slot_gb[s] << "ull), x); }\n";
    }
    os << "    }\n";
  }
  os << "    base = ((base | ~" << outer << ") + 1) & " << outer << ";\n"
     << (sp.pipe ? "    cur ^= " + std::to_string(tbytes) + "u;\n" : std::string());
  // smem reuse by the next tile (not needed when no round touches smem)
  const bool smem_used = !(d0.ok && dl.ok && nr == 1);
  if (smem_used) os << "    __syncthreads();\n";
  os << "  }\n";
  if (sp.check) os << "  if (__syncthreads_or(bad) && t == 0) atomicOr(flag, 1);\n";
  os << "}\n";
  return kPrelude + os.str();
}

std::string jit_key(const JitPassSpec& sp, const MicroPass& mp) {
  // every input of jit_source, as bytes (exact: no hash collisions)
  std::string k;
  auto put = [&](const void* p, size_t n) { k.append(static_cast<const char*>(p), n); };
  const int32_t head[] = {sp.device, sp.debug, sp.k, sp.R, sp.check, sp.pipe, sp.pf_bits, sp.min_blocks, sp.ring, sp.kparam, sp.tma_store, sp.fuse_k, sp.fuse_v[0], sp.fuse_v[1], sp.fuse_v[2],
                          sp.coalesce_bits,
                          static_cast<int32_t>(sp.rounds.size()),
                          static_cast<int32_t>(sp.tile_phys.size()),
                          static_cast<int32_t>(mp.words.size()),
                          static_cast<int32_t>(mp.pool.size())};
  put(head, sizeof(head));
  put(&sp.ntiles, 8);
  put(&sp.lo_mask, 8);
  put(&sp.outer_mask, 8);
  put(sp.slot_gb, sizeof(sp.slot_gb));
  put(sp.slot_sb, sizeof(sp.slot_sb));
  put(sp.swzv, sizeof(sp.swzv));
  put(sp.rounds.data(), sp.rounds.size() * sizeof(DRound));
  put(sp.tile_phys.data(), sp.tile_phys.size() * sizeof(int));
  put(mp.round_first.data(), mp.round_first.size() * 2);
  put(mp.round_count.data(), mp.round_count.size() * 2);
  put(mp.words.data(), mp.words.size() * 4);
  put(mp.pool.data(), mp.pool.size() * 8);
  return k;
}

namespace {

// Loads a CUBIN and fills the launch facts; caller holds no lock.
CacheEntry load_entry(const std::vector<char>& bin, const JitPassSpec& sp,
                      const std::vector<double>& kparams) {
  CacheEntry e;
  if (!kparams.empty()) e.k.kp = std::make_shared<const std::vector<double>>(kparams);
  if (cudaLibraryLoadData(&e.lib, bin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
      cudaLibraryGetKernel(&e.k.fn, e.lib, "qtjit") != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error("loading a compiled pass failed");
  }
  e.k.fuse_k = sp.fuse_k;
  e.k.threads = (sp.ring ? 2 : 1) << (sp.k - sp.R);
  e.k.smem = sp.ring ? 3 * (sizeof(double2) << sp.k) + 64 : (sp.pipe ? 2 : 1) * (sizeof(double2) << sp.k);
  // warp-staged drain: 2 KiB per warp after the mbarriers (jit_source_ring stage_off)
  if (sp.ring && sp.tma_store == 2)
    e.k.smem = 3 * (sizeof(double2) << sp.k) + 1024 + (static_cast<size_t>(2) << (sp.k - sp.R)) / 32 * 2048;
  const void* fn = reinterpret_cast<const void*>(e.k.fn);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(e.k.smem)) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&e.k.occupancy, fn, e.k.threads, e.k.smem) !=
          cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error("compiled pass: attribute / occupancy query failed");
  }
  e.k.occupancy = std::max(1, e.k.occupancy);
  return e;
}

// ---- background compiles (hybrid mode) --------------------------------------
struct Job {
  std::string key;
  JitPassSpec spec;
  MicroPass mp;  // the source is generated on the worker (off the caller's path)
  int device;
};
// heap-allocated and never destroyed: the detached workers may still wait on
// them while the process exits
std::mutex& q_mu = *new std::mutex();
std::condition_variable& q_cv = *new std::condition_variable();
std::deque<Job>* g_queue = nullptr;
std::unordered_map<std::string, int>* g_queued = nullptr;  // keys queued or compiling
int g_workers = 0;
int g_active = 0;       // jobs being compiled / loaded
bool g_exiting = false;
unsigned g_reregs = 0;  // background compiles finished (drain re-registration)

// At exit: drop the queue and wait for the jobs in flight, so no worker is
// inside NVRTC or the CUDA runtime while the runtime tears down.
bool g_trace = false;  // QTB_SEGV_TRACE: log the drain

void drain_at_exit() {
  std::unique_lock<std::mutex> lk(q_mu);
  g_exiting = true;
  if (g_trace) std::fprintf(stderr, "qtask-b200: exit drain: %d active, %zu queued\n", g_active, g_queue->size());
  g_queue->clear();
  q_cv.wait_for(lk, std::chrono::seconds(60), [] { return g_active == 0; });
  if (g_trace) std::fprintf(stderr, "qtask-b200: exit drain done (%d active)\n", g_active);
}

void worker() {
  for (;;) {
    Job j;
    {
      std::unique_lock<std::mutex> lk(q_mu);
      q_cv.wait(lk, [] { return !g_queue->empty() && !g_exiting; });
      j = std::move(g_queue->front());
      g_queue->pop_front();
      ++g_active;
    }
    const auto t0 = std::chrono::steady_clock::now();
    try {
      std::vector<double> kp;
      const std::vector<char> bin = compile_cubin(jit_source(j.spec, j.mp, &kp));
      cudaSetDevice(j.device);
      CacheEntry e = load_entry(bin, j.spec, kp);
      std::lock_guard<std::mutex> lk(g_mu);
      cache().emplace(j.key, e);
      ++g_stats.compiled;
      ++g_stats.background;
      g_stats.compile_ms +=
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    } catch (const std::exception&) {
      std::lock_guard<std::mutex> lk(g_mu);
      ++g_stats.failed;  // that pass keeps running on the interpreter
    }
    std::lock_guard<std::mutex> lk(q_mu);
    g_queued->erase(j.key);
    --g_active;
    // NVRTC may register more exit-time destructors lazily (new code paths
    // in a compile); re-registering the drain after a compile keeps it ahead
    // of them in the (reverse-order) exit sequence
    if (!g_exiting && (g_reregs < 64 || (g_reregs & 15) == 0)) std::atexit(drain_at_exit);
    ++g_reregs;
    q_cv.notify_all();
  }
}

}  // namespace

std::vector<JitKernel> jit_kernels(const std::vector<std::string>& keys,
                                   const std::vector<std::function<std::string(std::vector<double>*)>>& sources,
                                   const std::vector<JitPassSpec*>& specs) {
  std::vector<JitKernel> out(keys.size());
  std::vector<size_t> todo;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i = 0; i < keys.size(); ++i) {
      auto it = cache().find(keys[i]);
      if (it != cache().end()) {
        out[i] = it->second.k;
        ++g_stats.cache_hits;
      } else {
        todo.push_back(i);
      }
    }
  }
  if (todo.empty()) return out;
  const auto t0 = std::chrono::steady_clock::now();
  // parallel NVRTC compiles (independent programs)
  std::vector<std::vector<char>> bins(keys.size());
  std::vector<std::vector<double>> kps(keys.size());
  const size_t nthr = std::max<size_t>(1, std::min<size_t>(todo.size(), std::thread::hardware_concurrency()));
  std::atomic<size_t> next{0};
  std::mutex err_mu;
  std::string err;
  struct Ctx {
    std::function<void()> fn;
  } ctx{[&] {
    for (size_t j; (j = next.fetch_add(1)) < todo.size();) {
      try {
        bins[todo[j]] = compile_cubin(sources[todo[j]](&kps[todo[j]]));
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(err_mu);
        if (err.empty()) err = e.what();
      }
    }
  }};
  std::vector<pthread_t> ths;
  for (size_t w = 0; w < nthr; ++w) {
    pthread_attr_t attr;
    pthread_attr_init(&attr);
    pthread_attr_setstacksize(&attr, kJitStackBytes);
    pthread_t th;
    if (pthread_create(&th, &attr, [](void* c) -> void* { static_cast<Ctx*>(c)->fn(); return nullptr; },
                       &ctx) == 0)
      ths.push_back(th);
    pthread_attr_destroy(&attr);
  }
  if (ths.empty()) ctx.fn();
  for (pthread_t th : ths) pthread_join(th, nullptr);
  if (!err.empty()) throw std::runtime_error(err);
  for (size_t i : todo) {
    CacheEntry e = load_entry(bins[i], *specs[i], kps[i]);
    out[i] = e.k;
    std::lock_guard<std::mutex> lk(g_mu);
    cache().emplace(keys[i], e);
    ++g_stats.compiled;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_stats.compile_ms +=
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

bool jit_lookup(const std::string& key, JitKernel* out) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = cache().find(key);
  if (it == cache().end()) {
    ++g_stats.misses;
    return false;
  }
  *out = it->second.k;
  ++g_stats.cache_hits;
  return true;
}

void jit_compile_async(const std::string& key, const JitPassSpec& spec, const MicroPass& mp,
                       int device) {
  static std::once_flag first;
  std::call_once(first, [&] {
    // The first pass compiles synchronously, BEFORE the exit drain is
    // registered: NVRTC registers exit-time destructors lazily during its
    // first compile, and exit handlers run in reverse order -- ours must run
    // first, so that no background compile is still inside NVRTC when its
    // state is torn down.
    const auto t0 = std::chrono::steady_clock::now();
    try {
      std::vector<double> kp;
      const std::vector<char> bin = compile_cubin(jit_source(spec, mp, &kp));
      CacheEntry e = load_entry(bin, spec, kp);
      std::lock_guard<std::mutex> lk(g_mu);
      cache().emplace(key, e);
      ++g_stats.compiled;
      g_stats.compile_ms +=
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    } catch (const std::exception&) {
      std::lock_guard<std::mutex> lk(g_mu);
      ++g_stats.failed;
    }
    std::lock_guard<std::mutex> lk(q_mu);
    g_queue = new std::deque<Job>();
    g_queued = new std::unordered_map<std::string, int>();
    if (const char* e = std::getenv("QTB_SEGV_TRACE")) g_trace = std::atoi(e) != 0;
    std::atexit(drain_at_exit);
  });
  std::lock_guard<std::mutex> lk(q_mu);
  {
    std::lock_guard<std::mutex> lk2(g_mu);
    if (cache().count(key)) return;  // (the synchronous first compile)
  }
  if (g_exiting) return;
  if (g_queued->count(key)) return;
  (*g_queued)[key] = 1;
  // newest first (the latest edits' passes are the likeliest to recur), and a
  // bounded backlog: under a stream of edits the oldest queued passes are
  // dropped rather than compiled late
  g_queue->push_front(Job{key, spec, mp, device});
  while (g_queue->size() > kJitMaxBacklog) {
    g_queued->erase(g_queue->back().key);
    g_queue->pop_back();
  }
  if (g_workers < kJitBackgroundThreads) {
    ++g_workers;
    // NVRTC recurses deeply on long straight-line kernels: give the
    // compile threads a large stack (the default 8 MB can overflow)
    pthread_attr_t attr;
    pthread_attr_init(&attr);
    pthread_attr_setstacksize(&attr, kJitStackBytes);
    pthread_attr_setdetachstate(&attr, PTHREAD_CREATE_DETACHED);
    pthread_t th;
    if (pthread_create(&th, &attr, [](void*) -> void* { worker(); return nullptr; }, nullptr) != 0)
      --g_workers;
    pthread_attr_destroy(&attr);
  }
  q_cv.notify_all();
}

size_t jit_pending() {
  std::lock_guard<std::mutex> lk(q_mu);
  return g_queued ? g_queued->size() : 0;
}

cudaError_t jit_launch(const JitKernel& k, uint64_t ntiles, int sms, double2* psi,
                       const double2* src, int* flag, uint64_t gbase_hi, cudaStream_t s,
                       const JitFuseParams* fuse) {
  if ((k.fuse_k > 0) != (fuse != nullptr)) return cudaErrorInvalidValue;
  const uint64_t cap = static_cast<uint64_t>(k.occupancy) * static_cast<uint64_t>(sms);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(ntiles, cap));
  uint64_t per = (ntiles + grid - 1) / grid;
  // parameter 6 is the constant block (kparam passes) or the fused-exchange
  // table (never both: fused passes keep their constants as literals)
  void* args[] = {&psi, &src, &flag, &gbase_hi, &per,
                  fuse ? const_cast<JitFuseParams*>(fuse)
                       : (k.kp ? static_cast<void*>(const_cast<double*>(k.kp->data())) : nullptr)};
  return cudaLaunchKernel(reinterpret_cast<const void*>(k.fn), dim3(grid), dim3(k.threads), args,
                          k.smem, s);
}

bool jit_available(std::string* why) {
  const Nvrtc& n = nvrtc();
  if (why) *why = n.why;
  return n.ok;
}

std::vector<char> jit_compile_cubin(const std::string& src) { return compile_cubin(src); }

JitStats jit_stats() {
  std::lock_guard<std::mutex> lk(g_mu);
  JitStats st = g_stats;
  st.disk_hits = g_disk_hits.load();
  st.disk_writes = g_disk_writes.load();
  return st;
}

}  // namespace qtb

// ---- diagnostics: QTB_SEGV_TRACE=1 prints a native backtrace on SIGSEGV ----
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>
namespace {
void segv_trace(int sig) {
  void* bt[64];
  const int n = backtrace(bt, 64);
  const char msg[] = "qtask-b200: fatal signal, native backtrace:\n";
  (void)!write(2, msg, sizeof(msg) - 1);
  backtrace_symbols_fd(bt, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
struct SegvTraceInit {
  SegvTraceInit() {
    if (const char* e = std::getenv("QTB_SEGV_TRACE"))
      if (std::atoi(e) != 0) signal(SIGSEGV, segv_trace);
  }
} g_segv_trace_init;
}  // namespace
