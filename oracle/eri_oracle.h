/* oracle/eri_oracle.h — CPU restatement of the reference's Fock-build path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker. The product (paper_2412_13203_b200/) never links it.
 *
 * Every function restates reference behaviour and cites it; the restatement
 * is pinned against oracle/_ref (the unmodified reference headers compiled
 * here) by tests/test_oracle_pins.py and the committed fixtures in
 * tests/golden/.
 */
#ifndef ERI_ORACLE_H
#define ERI_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_ctx orc_ctx;

const char* orc_last_error(void);
/* parse_xyz (molecule.hpp:105-158) + BasisSetTable::parse (basis_set.hpp:33-84)
 * + attach_basis (basis_set.hpp:127-155) + build_pairs (block.hpp:52-103)
 * + tile_pairs (block.hpp:115-131) + make_blocks (block.hpp:145-150). */
orc_ctx* orc_create(const char* xyz_text, const char* basis_text, double kappa_screen,
                    int tile_size);
void orc_destroy(orc_ctx* c);
int orc_nbf(orc_ctx* c);
int orc_nshells(orc_ctx* c);
int orc_npairs(orc_ctx* c);
int orc_ntiles(orc_ctx* c);
long long orc_nblocks(orc_ctx* c);
int orc_natoms(orc_ctx* c);
int orc_nelectrons(orc_ctx* c);
void orc_atoms(orc_ctx* c, int* Z, double* pos);
void orc_shells(orc_ctx* c, int* L, int* K, int* atom, int* bf_off, double* center);
void orc_shell_prims(orc_ctx* c, int s, double* exps, double* coefs);
void orc_pairs(orc_ctx* c, int* i, int* j, int* nprim);
void orc_pair_prims(orc_ctx* c, int x, double* rec /* nprim x 13 */);
void orc_tiles(orc_ctx* c, int* li, int* lj, int* first, int* count);

/* boys_inplace (boys.hpp:23-44). */
void orc_boys(int m, double T, double* F);
/* Scaled integrals of one quartet, a-major over (i,j,k,l) components. */
int orc_eri_quartet(orc_ctx* c, int x, int y, double* out);
/* Schwarz Q per pair, pair-store order (rule: DESIGN.md "Screening"). */
int orc_schwarz(orc_ctx* c, double* Q);
void orc_set_schwarz(orc_ctx* c, const double* Q);
/* Canonical screened quartets x<=y in pair-store indices, block order. */
long long orc_quartets(orc_ctx* c, double tau, int* xs, int* ys, long long cap);
/* True J and K, tau<=0 disables screening. */
int orc_build_jk(orc_ctx* c, const double* D, double tau, int nthreads, double* J, double* K,
                 long long* nquartets);
int orc_build_jk_sample(orc_ctx* c, const double* D, double tau, int nthreads,
                        long long stride, long long offset, double* J, double* K,
                        long long* nquartets);
/* As build_jk_sample; *seconds = wall time of the parallel ERI+digestion
 * phase only (excludes partial-matrix allocation and merge). */
int orc_build_jk_timed(orc_ctx* c, const double* D, double tau, int nthreads, long long stride,
                       long long offset, double* J, double* K, long long* nquartets, double* seconds);
/* D-sparse build: as build_jk, but quartets whose six D blocks are all zero
 * are skipped (their contributions are exactly zero); *nquartets counts the
 * evaluated ones. Makes full-size parity checks cheap with a sparse D. */
int orc_build_jk_dsparse(orc_ctx* c, const double* D, double tau, int nthreads, double* J,
                         double* K, long long* nquartets);
/* J/K over an explicit canonical quartet list (x <= y, pair-store indices). */
int orc_build_jk_list(orc_ctx* c, const double* D, long long n, const int* xs, const int* ys,
                      int nthreads, double* J, double* K);
/* Per pair x: surviving canonical quartets (x, y >= x) and the wrapping sum
 * of splitmix64(y) over them; returns the total. */
long long orc_pair_survivors(orc_ctx* c, double tau, long long* count, unsigned long long* ysum);
/* One-electron S, T, V, McMurchie-Davidson; scaled. */
int orc_one_electron(orc_ctx* c, double* S, double* T, double* V);
double orc_nuclear_repulsion(orc_ctx* c);

#ifdef __cplusplus
}
#endif
#endif
