/* oracle/cg_oracle.h -- TEST INFRASTRUCTURE: plain-C FP64 restatement of the
 * reference hot path, used only by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the CHECKER.  Never linked into the product.
 *
 * Same batch layout and status bits as oracle/ref_shim.cpp (see there).
 * Pinned against oracle/_ref (the reference itself) and tests/golden/.
 */
#ifndef CG_ORACLE_H
#define CG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int orc_constellation(int qam_bits, double* points, double* axis0, double* axis1);
int orc_compute_llrs(double xr, double xi, double mu, double rho, int qam_bits, double* out);

int orc_detect_cg(int B, int U, long n_sc, int S, const double* H, const double* Y,
                  double rho_u, double n0, double es, int qam_bits, int K, int tracker,
                  double* xhat, double* mu, double* rho, double* llr, uint8_t* status);
int orc_detect_explicit(int B, int U, long n_sc, int S, const double* H, const double* Y,
                        double rho_u, double n0, double es, int qam_bits, double* xhat,
                        double* mu, double* rho, double* llr, uint8_t* status);
int orc_precode_cg(int B, int U, long n_sc, int S, const double* Hd, const double* T,
                   double rho_d, int K, double* q, double* s, double* gain, uint8_t* status);
int orc_precode_explicit(int B, int U, long n_sc, int S, const double* Hd, const double* T,
                         double rho_d, double* q, double* s, double* gain, uint8_t* status);

/* the trade-off study's other solvers (detect.cpp:122-326, precode.cpp:45-93) */
int orc_detect_cholesky(int B, int U, long n_sc, int S, const double* H, const double* Y,
                        double rho_u, double n0, double es, int qam_bits, double* xhat,
                        double* mu, double* rho, double* llr, uint8_t* status);
int orc_detect_cgls(int B, int U, long n_sc, int S, const double* H, const double* Y,
                    double rho_u, double n0, double es, int qam_bits, int K, double* xhat,
                    double* mu, double* rho, double* llr, uint8_t* status);
int orc_detect_neumann(int B, int U, long n_sc, int S, const double* H, const double* Y,
                       double rho_u, double n0, double es, int qam_bits, int K, double* xhat,
                       double* mu, double* rho, double* llr, uint8_t* status);
int orc_precode_cgls(int B, int U, long n_sc, int S, const double* Hd, const double* T,
                     double rho_d, int K, double* q, double* s, double* gain, uint8_t* status);
int orc_precode_neumann(int B, int U, long n_sc, int S, const double* Hd, const double* T,
                        double rho_d, int K, double* q, double* s, double* gain, uint8_t* status);

void orc_rng_u64(uint64_t key, const uint64_t* forks, int n_forks, long n, uint64_t* out);
void orc_rng_cgaussian(uint64_t key, const uint64_t* forks, int n_forks, double variance,
                       long n, double* out);
void orc_rayleigh(uint64_t key, const uint64_t* forks, int n_forks, int B, int U, double* out);

/* coded BLER harness (coding.cpp): same contracts as the ref_ entry points in
 * ref_shim.cpp -- lengths returned, -1 on a length the reference rejects */
long orc_conv_encode(const uint8_t* info, long n, uint8_t* out);
long orc_viterbi_decode(const double* llrs, long n, uint8_t* out);
void orc_make_interleaver(uint64_t key, const uint64_t* forks, int n_forks, long n, int64_t* perm);

#ifdef __cplusplus
}
#endif
#endif
