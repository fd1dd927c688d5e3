// tests/dropin/relink_sim_main.cpp -- TEST INFRASTRUCTURE.
//
// The reference's OWN caller of the hot path, relinked: sim::run_uplink_sweep
// and sim::run_downlink_sweep (/root/reference/proj/src/sim.cpp:147-405; its
// equalize / run_precoder call detect::detect_cg and precode::precode_cg per
// (symbol, subcarrier), sim.cpp:120-145) compiled from the unmodified
// reference sources and headers, linked against libcgmimo_b200.so for every
// detect:: / precode:: entry point, the constellation tables and the opcount
// hooks instead of the reference's detect.cpp / precode.cpp / solvers.cpp /
// constellation.cpp (oracle/Makefile target `relink`).  Prints one line per
// sweep point: direction snr frames block_errors breakdowns trials.
#include <cstdio>
#include <cstdlib>

#include "cgmimo/sim.hpp"

using namespace cgmimo;

int main(int argc, char** argv) {
  const int tracker = argc > 1 ? std::atoi(argv[1]) : 1;
  sim::SweepConfig cfg;
  cfg.bs_antennas = 32;
  cfg.users = 8;
  cfg.modulation = phy::Modulation::kQam64;
  cfg.method = sim::Method::kCg;
  cfg.iterations = 4;
  cfg.tracker = tracker == 0 ? detect::SinrTracker::kExact : detect::SinrTracker::kApprox;
  cfg.snr_start_db = 12.0;
  cfg.snr_stop_db = 14.0;
  cfg.snr_step_db = 2.0;
  cfg.trials = 12;
  cfg.subcarriers = 16;
  cfg.seed = 7;
  cfg.threads = 4;
  cfg.max_breakdown_fraction = 1.0;
  for (int dir = 0; dir < 2; ++dir) {
    const sim::SweepResult r = dir == 0 ? sim::run_uplink_sweep(cfg) : sim::run_downlink_sweep(cfg);
    for (const auto& pt : r.points)
      std::printf("%s %.1f %llu %llu %llu %llu\n", dir == 0 ? "uplink" : "downlink", pt.snr_db,
                  static_cast<unsigned long long>(pt.frames),
                  static_cast<unsigned long long>(pt.block_errors),
                  static_cast<unsigned long long>(pt.breakdowns),
                  static_cast<unsigned long long>(pt.trials_run));
  }
  return 0;
}
