// schedule_check.cpp -- host-side proof for the single-kernel FFT schedules.
//
// For a configuration (m, LOG_E, W, stage split) this program
//  1. replays the kernel's schedule (csrc/schedule.cuh) symbolically and checks
//     that every butterfly matches the reference dataflow of run_passes
//     (fft.cpp:32-52): same two operand positions, same operand order, same
//     table entry, same two output positions; and that the final buffer is in
//     natural order;
//  2. counts shared-memory wavefronts of every warp-wide access the kernel
//     issues (identity loads/stores, padded exchange, twiddle records) against
//     the conflict-free ideal.
//
//   g++ -O2 -std=c++17 -I paper_2604_00567_b200/csrc tools/schedule_check.cpp
//   ./a.out [m logE W s0 s1 ...]       (no args: sweep the shipped configs)
#include <cstdio>
#include <functional>
#include <algorithm>
#include <cstdlib>
#include <map>
#include <set>
#include <tuple>
#include <vector>

#include "schedule.cuh"

using namespace dsfft;

struct Cfg {
  int m, logE, W;
  std::vector<int> s;
  int fp16;  // 0 fp32; 1 fp16 transform pairs (identity 2 x half2); 2 fp16 complex (4-byte values)
};

// Wavefronts for one warp access: addr[lane] byte address, B bytes per lane.
static int wavefronts(const std::vector<long>& addr, int B) {
  const int lanes_per_phase = 128 / B < 32 ? 128 / B : 32;
  int total = 0;
  for (int p0 = 0; p0 < 32; p0 += lanes_per_phase) {
    std::map<int, std::set<long>> bank_words;
    for (int l = p0; l < p0 + lanes_per_phase; ++l) {
      if (addr[l] < 0) continue;
      for (int w = 0; w < B / 4; ++w) {
        long word = addr[l] / 4 + w;
        bank_words[int(word % 32)].insert(word);
      }
    }
    int deg = 0;
    for (auto& kv : bank_words) deg = std::max<int>(deg, int(kv.second.size()));
    total += deg ? deg : 0;
  }
  return total;
}

struct Tally {
  long ideal = 0, actual = 0;
  void add(const std::vector<long>& a, int B) {
    ideal += (B * 32 + 127) / 128;
    actual += wavefronts(a, B);
  }
};

static bool check(const Cfg& c, bool verbose) {
  const int m = c.m, N = 1 << m, E = 1 << c.logE, T = 32 * c.W;
  const int VALS = T * E;
  if (VALS % N) { printf("bad: VALS %% N\n"); return false; }
  const int K = VALS / N;
  int sum = 0;
  for (int s : c.s) { if (s > c.logE || s < 1) return false; sum += s; }
  if (sum != m) return false;

  // --- 1. symbolic dataflow ------------------------------------------------
  // label = position after `pass` passes; buffer holds labels (k, pass, pos).
  struct Lab { int k, pass, pos; };
  std::vector<Lab> buf(VALS);
  for (int k = 0; k < K; ++k)
    for (int p = 0; p < N; ++p) buf[k * N + p] = {k, 0, p};
  bool ok = true;
  int P = 0;
  for (size_t st = 0; st < c.s.size(); ++st) {
    const int s = c.s[st];
    std::vector<Lab> nb(VALS, Lab{-1, -1, -1});
    for (int t = 0; t < T; ++t) {
      for (int j = 0; j < (E >> s); ++j) {
        const int G = t + T * j;
        std::vector<Lab> v(1 << s);
        for (int cc = 0; cc < (1 << s); ++cc) v[cc] = buf[read_pos(m, P, s, G, cc)];
        const int r = grp_r(m, P, s, G);
        for (int pl = 0; pl < s; ++pl) {
          std::vector<Lab> w(1 << s);
          for (int jl = 0; jl < (1 << (s - 1)); ++jl) {
            const int rl = jl & ((1 << pl) - 1);
            const Lab a = v[jl], b = v[jl + (1 << (s - 1))];
            const int p = P + pl;
            // reference butterfly j = a.pos at pass p
            const int jr = a.pos, block = 1 << p;
            const bool good = a.pass == p && b.pass == p && a.k == b.k && jr < N / 2 &&
                              b.pos == jr + N / 2 &&
                              tw_entry(m, P, r, pl, rl) == (jr & (block - 1)) * (N / (2 * block));
            if (!good) {
              if (verbose) printf("  dataflow mismatch stage %zu pl %d\n", st, pl);
              ok = false;
            }
            const int base = ((jr >> p) * 2) * block + (jr & (block - 1));
            w[(jl >> pl) * (2 << pl) + rl] = {a.k, p + 1, base};
            w[(jl >> pl) * (2 << pl) + rl + (1 << pl)] = {a.k, p + 1, base + block};
          }
          v = w;
        }
        for (int cc = 0; cc < (1 << s); ++cc) {
          const int wp = write_pos(m, P, s, G, cc);
          if (v[cc].pos != wp % N || v[cc].k != wp / N || v[cc].pass != P + s) ok = false;
          if (nb[wp].pass != -1) ok = false;  // double write
          nb[wp] = v[cc];
        }
      }
    }
    buf = nb;
    P += s;
  }
  for (int k = 0; k < K; ++k)
    for (int p = 0; p < N; ++p)
      if (buf[k * N + p].pass != m || buf[k * N + p].pos != p || buf[k * N + p].k != k) ok = false;

  // --- 2. bank conflicts (per warp 0..W-1, every access) -----------------
  Tally ld, ex_w, ex_r, stv, tw;
  const int VB = c.fp16 == 2 ? 4 : 8;  // exchange value bytes
  P = 0;
  const int nst = int(c.s.size());
  for (int st = 0; st < nst; ++st) {
    const int s = c.s[st];
    for (int w = 0; w < c.W; ++w) {
      for (int j = 0; j < (E >> s); ++j) {
        for (int cc = 0; cc < (1 << s); ++cc) {
          std::vector<long> ar(32), aw(32), ar1(32), aw1(32);
          for (int l = 0; l < 32; ++l) {
            const int G = 32 * w + l + T * j;
            const int rp = read_pos(m, P, s, G, cc), wp = write_pos(m, P, s, G, cc);
            if (c.fp16 == 1) {
              // identity: real transform 2k+h, half2 (4 bytes)
              ar[l] = long((2 * (rp / N)) * N + rp % N) * 4;
              ar1[l] = long((2 * (rp / N) + 1) * N + rp % N) * 4;
              aw[l] = long((2 * (wp / N)) * N + wp % N) * 4;
              aw1[l] = long((2 * (wp / N) + 1) * N + wp % N) * 4;
            } else {
              ar[l] = long(rp) * VB;
              aw[l] = long(wp) * VB;
            }
          }
          const int IB = c.fp16 ? 4 : 8;  // identity access width
          if (st == 0) { ld.add(ar, IB); if (c.fp16 == 1) ld.add(ar1, 4); }
          else {
            std::vector<long> a(32);
            for (int l = 0; l < 32; ++l)
              a[l] = long(pad_pos(read_pos(m, P, s, 32 * w + l + T * j, cc))) * VB;
            ex_r.add(a, VB);
          }
          if (st == nst - 1) { stv.add(aw, IB); if (c.fp16 == 1) stv.add(aw1, 4); }
          else {
            std::vector<long> a(32);
            for (int l = 0; l < 32; ++l)
              a[l] = long(pad_pos(write_pos(m, P, s, 32 * w + l + T * j, cc))) * VB;
            ex_w.add(a, VB);
          }
        }
        // twiddles: one LDS.128 per (pl, rl)
        for (int pl = 0; pl < s; ++pl)
          for (int rl = 0; rl < (1 << pl); ++rl) {
            std::vector<long> a(32);
            for (int l = 0; l < 32; ++l)
              a[l] = long(tw_slot(P, grp_r(m, P, s, 32 * w + l + T * j), pl, rl)) * 16;
            tw.add(a, 16);
          }
      }
    }
    P += s;
  }
  printf("m=%2d logE=%d W=%d %s stages=", m, c.logE, c.W, c.fp16 == 2 ? "f16c" : c.fp16 ? "f16p" : "fp32");
  for (int s : c.s) printf("%d ", s);
  printf("| dataflow %s | wavefronts actual/ideal: load %ld/%ld exw %ld/%ld exr %ld/%ld "
         "store %ld/%ld tw %ld/%ld\n",
         ok ? "OK " : "BAD", ld.actual, ld.ideal, ex_w.actual, ex_w.ideal, ex_r.actual,
         ex_r.ideal, stv.actual, stv.ideal, tw.actual, tw.ideal);
  return ok;
}

int main(int argc, char** argv) {
  if (argc > 4) {
    Cfg c{atoi(argv[1]), atoi(argv[2]), atoi(argv[3]), {}, 0};
    for (int i = 4; i < argc; ++i) c.s.push_back(atoi(argv[i]));
    c.fp16 = 0;
    bool ok = check(c, true);
    c.fp16 = 1;
    ok = check(c, true) && ok;
    c.fp16 = 2;
    ok = check(c, true) && ok;
    return ok ? 0 : 1;
  }
  // sweep all stage splits for the single-kernel sizes
  int bad = 0;
  for (int m = 6; m <= 12; ++m)
    for (int logE = 4; logE <= 6; ++logE)
      for (int W = 1; W <= 4; W *= 2) {
        if ((32 * W << logE) < (1 << m)) continue;
        if ((32 * W << logE) > 4 * (1 << m) && m >= 10) continue;
        // enumerate compositions of m into parts <= logE, at most 4 parts
        std::vector<std::vector<int>> comps;
        std::vector<int> cur;
        std::function<void(int)> rec;
        (void)rec;
        for (int a = 1; a <= logE; ++a)
          for (int b = 0; b <= logE; ++b)
            for (int d = 0; d <= logE; ++d) {
              if (b == 0 && d) continue;
              if (a + b + d != m) continue;
              std::vector<int> v{a};
              if (b) v.push_back(b);
              if (d) v.push_back(d);
              comps.push_back(v);
            }
        for (auto& v : comps)
          for (int f = 0; f <= 2; ++f) {
            Cfg c{m, logE, W, v, f};
            if (!check(c, false)) ++bad;
          }
      }
  return bad ? 1 : 0;
}
