// A caller written against the reference's C++ API (cgmimo::detect /
// cgmimo::precode / cgmimo::phy / cgmimo::opcount), compiled against the
// drop-in headers in include/cgmimo/ and linked with libcgmimo_b200.so.
//   dropin_main host            : host-only checks, prints tables as text
//   dropin_main gpu in.bin out.bin : per-call detect_cg / precode_cg on the GPU
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <vector>

#include "cgmimo/constellation.hpp"
#include "cgmimo/detect.hpp"
#include "cgmimo/opcount.hpp"
#include "cgmimo/precode.hpp"
#include "cgmimo/solvers.hpp"

using namespace cgmimo;

static int host_mode() {
  for (auto m : {phy::Modulation::kQpsk, phy::Modulation::kQam16, phy::Modulation::kQam64}) {
    const auto c = phy::make_constellation(m);
    std::printf("constellation %d", c.bits_per_symbol);
    for (const auto& pt : c.points) std::printf(" %.17g %.17g", pt.real(), pt.imag());
    std::printf("\n");
    // map/demap round trip
    std::vector<std::uint8_t> bits;
    for (unsigned l = 0; l < c.points.size(); ++l)
      for (int b = 0; b < c.bits_per_symbol; ++b) bits.push_back((l >> (c.bits_per_symbol - 1 - b)) & 1u);
    const auto sym = phy::map_bits(bits, c);
    for (unsigned l = 0; l < sym.size(); ++l)
      if (phy::hard_demap(sym[l], c) != l) return 10;
  }
  const struct { double xr, xi, mu, rho; phy::Modulation m; } cases[] = {
      {0.9, 0.9, 1.0, 2.0, phy::Modulation::kQam16}, {0.0, 0.5, 1.0, 2.0, phy::Modulation::kQam16},
      {0.9, 0.9, 1e-14, 10.0, phy::Modulation::kQam16}, {0.3, -1.1, 0.8, 40.0, phy::Modulation::kQam64},
      {-0.2, 0.05, 1.2, -3.0, phy::Modulation::kQam64}, {1.0, 0.0, 1.0, 1.5, phy::Modulation::kQpsk}};
  for (const auto& t : cases) {
    const auto l = detect::compute_llrs(cplx(t.xr, t.xi), t.mu, t.rho, phy::make_constellation(t.m));
    std::printf("llr");
    for (double v : l) std::printf(" %.17g", v);
    std::printf("\n");
  }
  // argument errors surface before any device work (detect.cpp:186-188)
  try {
    (void)detect::detect_cg(ComplexMatrix(8, 4), ComplexVector(7), 1.0, 1.0, 1.0,
                            phy::make_constellation(phy::Modulation::kQam16), 2,
                            detect::SinrTracker::kExact);
    return 11;
  } catch (const std::invalid_argument&) {
  }
  try {
    (void)precode::precode_cg(ComplexMatrix(4, 8), ComplexVector(4), -1.0, 2);
    return 12;
  } catch (const std::invalid_argument&) {
  }
  if (opcount::counting_active()) return 13;
  opcount::Tally t;
  {
    opcount::ScopedTally s(t);
    if (!opcount::counting_active()) return 14;
  }
  {  // HermitianMatrix (reference linalg.hpp:42-65): packed lower triangle
    HermitianMatrix h(3);
    h.set(0, 0, cplx(2.0, 5.0));  // imaginary part dropped on the diagonal
    h.set(1, 0, cplx(1.0, -0.5));
    h.set(1, 1, 3.0);
    h.set(2, 0, cplx(0.25, 0.75));
    h.set(2, 1, cplx(-1.5, 2.0));
    h.set(2, 2, 4.0);
    const ComplexMatrix f = h.full();
    std::printf("hermitian");
    for (std::size_t i = 0; i < 3; ++i)
      for (std::size_t j = 0; j < 3; ++j) std::printf(" %.17g %.17g", f(i, j).real(), f(i, j).imag());
    std::printf(" %.17g %.17g\n", h.diag(0), h.real_diag()[2]);
    bool threw = false;
    try {
      h.set(0, 1, 1.0);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    std::printf("hermitian_upper_set_throws %d\n", threw ? 1 : 0);
  }
  std::printf("host ok\n");
  return 0;
}

// in.bin: int32 B, U, K, bits, tracker, n; then n x (H[B][U], y[B]) complex128;
// then precode: int32 Bd, Ud, Kd, nd; nd x (Hd[Ud][Bd], t[Ud]); double rho_u, n0, rho_d
static int gpu_mode(const char* in, const char* out) {
  std::ifstream f(in, std::ios::binary);
  auto rd = [&](void* p, size_t n) { f.read(static_cast<char*>(p), n); };
  int hdr[6];
  rd(hdr, sizeof hdr);
  const int B = hdr[0], U = hdr[1], K = hdr[2], bits = hdr[3], trk = hdr[4], n = hdr[5];
  std::vector<ComplexMatrix> hs;
  std::vector<ComplexVector> ys;
  for (int i = 0; i < n; ++i) {
    ComplexMatrix h(B, U);
    for (int b = 0; b < B; ++b) rd(h.row(b), sizeof(cplx) * U);
    ComplexVector y(B);
    rd(y.data(), sizeof(cplx) * B);
    hs.push_back(h);
    ys.push_back(y);
  }
  int ph[4];
  rd(ph, sizeof ph);
  const int Bd = ph[0], Ud = ph[1], Kd = ph[2], nd = ph[3];
  std::vector<ComplexMatrix> hds;
  std::vector<ComplexVector> ts;
  for (int i = 0; i < nd; ++i) {
    ComplexMatrix h(Ud, Bd);
    for (int u = 0; u < Ud; ++u) rd(h.row(u), sizeof(cplx) * Bd);
    ComplexVector t(Ud);
    rd(t.data(), sizeof(cplx) * Ud);
    hds.push_back(h);
    ts.push_back(t);
  }
  double prm[3];
  rd(prm, sizeof prm);
  const auto c = phy::make_constellation(bits == 2 ? phy::Modulation::kQpsk
                                                   : bits == 4 ? phy::Modulation::kQam16
                                                               : phy::Modulation::kQam64);
  std::ofstream o(out, std::ios::binary);
  auto wr = [&](const void* p, size_t nb) { o.write(static_cast<const char*>(p), nb); };
  for (int i = 0; i < n; ++i) {
    opcount::Tally tally;
    detect::SoftOutput r;
    {
      opcount::ScopedTally s(tally);
      r = detect::detect_cg(hs[i], ys[i], prm[0], prm[1], 1.0, c, K,
                            trk == 0 ? detect::SinrTracker::kExact : detect::SinrTracker::kApprox);
    }
    wr(r.xhat.data(), sizeof(cplx) * U);
    wr(r.mu.data(), sizeof(double) * U);
    wr(r.rho.data(), sizeof(double) * U);
    for (int u = 0; u < U; ++u) wr(r.llrs[u].data(), sizeof(double) * bits);
    std::uint64_t st[opcount::kStageCount];
    for (int s = 0; s < opcount::kStageCount; ++s) st[s] = tally.get(static_cast<opcount::Stage>(s));
    wr(st, sizeof st);
  }
  for (int i = 0; i < nd; ++i) {
    std::vector<ComplexVector> trace;
    const auto r = precode::precode_cg(hds[i], ts[i], prm[2], Kd, &trace);
    wr(r.precoded.data(), sizeof(cplx) * Bd);
    wr(r.transmit.data(), sizeof(cplx) * Bd);
    wr(&r.gain, sizeof(double));
    const double z = r.zero_input ? 1.0 : 0.0;
    wr(&z, sizeof(double));
    for (const auto& q : trace) wr(q.data(), sizeof(cplx) * Bd);
  }
  // a breakdown surfaces as solvers::SolverBreakdown (solvers.cpp:55-57)
  int broke = 0;
  try {
    ComplexMatrix h0(4, 8);
    ComplexVector t0(4, cplx(1.0, 0.0));
    (void)precode::precode_cg(h0, t0, 1e35, 2);
  } catch (const solvers::SolverBreakdown&) {
    broke = 1;
  }
  wr(&broke, sizeof broke);
  return 0;
}

// in.bin: int32 B, U, bits, n, K; n x (H[B][U], y[B]); int32 Bd, Ud, nd, Kd;
// nd x (Hd[Ud][Bd], t[Ud]); double rho_u, n0, rho_d.  Per instance and
// method (cholesky, cgls K, neumann K): xhat, mu, rho, llr, stage tally; per
// precoder instance and method (explicit, cgls Kd, neumann Kd): q, s, gain.
static int alt_mode(const char* in, const char* out) {
  std::ifstream f(in, std::ios::binary);
  auto rd = [&](void* p, size_t n) { f.read(static_cast<char*>(p), n); };
  int hdr[5];
  rd(hdr, sizeof hdr);
  const int B = hdr[0], U = hdr[1], bits = hdr[2], n = hdr[3], K = hdr[4];
  std::vector<ComplexMatrix> hs;
  std::vector<ComplexVector> ys;
  for (int i = 0; i < n; ++i) {
    ComplexMatrix h(B, U);
    for (int b = 0; b < B; ++b) rd(h.row(b), sizeof(cplx) * U);
    ComplexVector y(B);
    rd(y.data(), sizeof(cplx) * B);
    hs.push_back(h);
    ys.push_back(y);
  }
  int ph[4];
  rd(ph, sizeof ph);
  const int Bd = ph[0], Ud = ph[1], nd = ph[2], Kd = ph[3];
  std::vector<ComplexMatrix> hds;
  std::vector<ComplexVector> ts;
  for (int i = 0; i < nd; ++i) {
    ComplexMatrix h(Ud, Bd);
    for (int u = 0; u < Ud; ++u) rd(h.row(u), sizeof(cplx) * Bd);
    ComplexVector t(Ud);
    rd(t.data(), sizeof(cplx) * Ud);
    hds.push_back(h);
    ts.push_back(t);
  }
  double prm[3];
  rd(prm, sizeof prm);
  const auto c = phy::make_constellation(bits == 2 ? phy::Modulation::kQpsk
                                                   : bits == 4 ? phy::Modulation::kQam16
                                                               : phy::Modulation::kQam64);
  std::ofstream o(out, std::ios::binary);
  auto wr = [&](const void* p, size_t nb) { o.write(static_cast<const char*>(p), nb); };
  for (int i = 0; i < n; ++i)
    for (int m = 0; m < 3; ++m) {
      opcount::Tally tally;
      detect::SoftOutput r;
      {
        opcount::ScopedTally s(tally);
        r = m == 0   ? detect::detect_cholesky(hs[i], ys[i], prm[0], prm[1], 1.0, c)
            : m == 1 ? detect::detect_cgls(hs[i], ys[i], prm[0], prm[1], 1.0, c, K)
                     : detect::detect_neumann(hs[i], ys[i], prm[0], prm[1], 1.0, c, K);
      }
      wr(r.xhat.data(), sizeof(cplx) * U);
      wr(r.mu.data(), sizeof(double) * U);
      wr(r.rho.data(), sizeof(double) * U);
      for (int u = 0; u < U; ++u) wr(r.llrs[u].data(), sizeof(double) * bits);
      std::uint64_t st[opcount::kStageCount];
      for (int s = 0; s < opcount::kStageCount; ++s) st[s] = tally.get(static_cast<opcount::Stage>(s));
      wr(st, sizeof st);
    }
  for (int i = 0; i < nd; ++i)
    for (int m = 0; m < 3; ++m) {
      const auto r = m == 0   ? precode::precode_explicit(hds[i], ts[i], prm[2])
                     : m == 1 ? precode::precode_cgls(hds[i], ts[i], prm[2], Kd)
                              : precode::precode_neumann(hds[i], ts[i], prm[2], Kd);
      wr(r.precoded.data(), sizeof(cplx) * Bd);
      wr(r.transmit.data(), sizeof(cplx) * Bd);
      wr(&r.gain, sizeof(double));
    }
  // argument errors as the reference (detect.cpp:243-245)
  int bad = 0;
  try {
    (void)detect::detect_cgls(hs[0], ys[0], prm[0], prm[1], 1.0, c, 0);
  } catch (const std::invalid_argument&) {
    bad = 1;
  }
  wr(&bad, sizeof bad);
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 2 && std::strcmp(argv[1], "host") == 0) return host_mode();
  if (argc >= 4 && std::strcmp(argv[1], "alt") == 0) return alt_mode(argv[2], argv[3]);
  if (argc >= 4 && std::strcmp(argv[1], "gpu") == 0) return gpu_mode(argv[2], argv[3]);
  std::fprintf(stderr, "usage: dropin_main host | gpu in.bin out.bin\n");
  return 2;
}
