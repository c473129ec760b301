/* oracle/eri_oracle.c — CPU restatement of the reference Fock-build path.
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA product, never the thing
 * measured or shipped (see eri_oracle.h). Written from the reference's
 * semantics, not from its code; each function cites what it restates.
 * Pinned against oracle/_ref (unmodified reference headers) by
 * tests/test_oracle_pins.py and the fixtures in tests/golden/.
 *
 * Integrals: the recurrences of dag.hpp:119-173 (vertical relations on
 * transferred nodes [e0|f0]^(m) per primitive quartet, horizontal relations
 * on contracted values, compiler.hpp:206-224 partition), evaluated along a
 * fixed path (first non-zero Cartesian direction) instead of the greedy
 * Alg. 1 path — same mathematics, round-off-level differences only.
 */
#define _GNU_SOURCE
#include "eri_oracle.h"

#include <ctype.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#define ANG2BOHR 1.8897259886 /* molecule.hpp:16 */
#define MAXL 4                /* shells up to g */
#define MAXLT (4 * MAXL)      /* total momentum of a quartet */
#define NMOM (((MAXLT + 1) * (MAXLT + 2) * (MAXLT + 3)) / 6)

static __thread char g_err[512];
const char* orc_last_error(void) { return g_err; }
static void set_err(const char* m) { snprintf(g_err, sizeof g_err, "%s", m); }

/* ---------------------------------------------------------------- elements */
/* elements.hpp:12-15 */
static const char* ELEM[36] = {"H",  "He", "Li", "Be", "B",  "C",  "N",  "O",  "F",
                               "Ne", "Na", "Mg", "Al", "Si", "P",  "S",  "Cl", "Ar",
                               "K",  "Ca", "Sc", "Ti", "V",  "Cr", "Mn", "Fe", "Co",
                               "Ni", "Cu", "Zn", "Ga", "Ge", "As", "Se", "Br", "Kr"};
/* elements.hpp:17-26 */
static int atomic_number_of(const char* sym) {
  char s[8];
  size_t n = strlen(sym);
  if (n == 0 || n > 6) return 0;
  for (size_t i = 0; i < n; ++i)
    s[i] = (char)(i ? tolower((unsigned char)sym[i]) : toupper((unsigned char)sym[i]));
  s[n] = 0;
  for (int z = 0; z < 36; ++z)
    if (strcmp(ELEM[z], s) == 0) return z + 1;
  return 0;
}

/* ------------------------------------------------------------------ types */
typedef struct {
  double c[3];
  int L, K, atom;
  double* exps;
  double* coefs;
} shell_t;

typedef struct { /* block.hpp:16-24 */
  double p, inv_two_p, P[3], PA[3], PB[3], kappa, coef;
} prim_t;

typedef struct { /* block.hpp:26-31 */
  int i, j, li, lj;
  double AB[3];
  int nprim;
  prim_t* prims;
} pair_t;

typedef struct {
  int li, lj, first, count;
} tile_t;
typedef struct {
  int bt, kt;
} block_t;

struct orc_ctx {
  int natoms, *Z;
  double* pos;
  int nshell;
  shell_t* sh;
  int* bf_off;
  int nbf;
  int npair;
  pair_t* pr;
  int ntile;
  tile_t* tl;
  long long nblock;
  block_t* bl;
  double* Q;
  int have_q;
};

/* ------------------------------------------------------- cartesian tables */
/* Momenta of total n in shell_components order (molecule.hpp:176-183):
 * ax descending, then ay descending. Global index = cart_off(n) + local. */
static int cart_off(int n) { return n * (n + 1) * (n + 2) / 6; }
static int ncart(int n) { return (n + 1) * (n + 2) / 2; }
static int g_mom[NMOM][3];
static int g_idx[MAXLT + 1][MAXLT + 1][MAXLT + 1];
static pthread_once_t g_once = PTHREAD_ONCE_INIT;
static void init_tables(void) {
  int g = 0;
  for (int n = 0; n <= MAXLT; ++n)
    for (int ax = n; ax >= 0; --ax)
      for (int ay = n - ax; ay >= 0; --ay) {
        g_mom[g][0] = ax;
        g_mom[g][1] = ay;
        g_mom[g][2] = n - ax - ay;
        g_idx[ax][ay][n - ax - ay] = g;
        ++g;
      }
}
static int idx3(int x, int y, int z) { return g_idx[x][y][z]; }

/* odd_double_factorial (molecule.hpp:199-203) */
static double odf(int n) {
  double v = 1.0;
  for (int k = 2 * n - 1; k > 1; k -= 2) v *= k;
  return v;
}
/* component_norm_scale (molecule.hpp:207-213) */
static double comp_scale(const int* m) {
  int L = m[0] + m[1] + m[2];
  if (L <= 1) return 1.0;
  return sqrt(odf(L) / (odf(m[0]) * odf(m[1]) * odf(m[2])));
}

/* ------------------------------------------------------------------ boys */
/* boys_inplace (boys.hpp:23-44), restated operation for operation. */
void orc_boys(int m_max, double T, double* F) {
  const double expT = exp(-T);
  if (T < 35.0 || 2 * m_max + 1 >= T) {
    double term = 1.0 / (2 * m_max + 1);
    double sum = term;
    for (int k = 0; term > 1e-17 * sum && k < 10000; ++k) {
      term *= 2.0 * T / (2 * m_max + 2 * k + 3);
      sum += term;
    }
    F[m_max] = expT * sum;
    for (int m = m_max; m > 0; --m) F[m - 1] = (2.0 * T * F[m] + expT) / (2 * m - 1);
  } else {
    const double sqrtT = sqrt(T);
    F[0] = 0.5 * sqrt(M_PI / T) * erf(sqrtT);
    for (int m = 0; m < m_max; ++m) F[m + 1] = ((2 * m + 1) * F[m] - expT) / (2.0 * T);
  }
}

/* --------------------------------------------------------------- parsing */
static char* dup_str(const char* s) {
  size_t n = strlen(s);
  char* d = malloc(n + 1);
  memcpy(d, s, n + 1);
  return d;
}
static char* next_line(char** cur) {
  if (!*cur || !**cur) return NULL;
  char* s = *cur;
  char* e = strchr(s, '\n');
  if (e) {
    *e = 0;
    *cur = e + 1;
  } else {
    *cur = s + strlen(s);
  }
  return s;
}
static char* trim(char* s) {
  while (*s && isspace((unsigned char)*s)) ++s;
  char* e = s + strlen(s);
  while (e > s && isspace((unsigned char)e[-1])) --e;
  *e = 0;
  return s;
}
static int parse_num(const char* tok, double* v) {
  char* end;
  *v = strtod(tok, &end);
  return *end == 0 && isfinite(*v);
}

typedef struct {
  int L, K;
  double *e, *c;
} rec_shell;
typedef struct {
  int n;
  rec_shell* s;
} rec_elem;

/* BasisSetTable::parse (basis_set.hpp:33-84) */
static int parse_basis(const char* text, rec_elem* tab /* [37] */) {
  char* buf = dup_str(text);
  char* cur = buf;
  char* line;
  int current = 0;
  while ((line = next_line(&cur))) {
    char* t = trim(line);
    if (!*t || t[0] == '#') continue;
    char head[64];
    if (sscanf(t, "%63s", head) != 1) continue;
    if (strcmp(head, "element") == 0) {
      char sym[16];
      if (sscanf(t, "%*s %15s", sym) != 1 || !(current = atomic_number_of(sym))) {
        set_err("basis: bad element record");
        free(buf);
        return -1;
      }
    } else {
      int L, K;
      if (!current || sscanf(t, "%d %d", &L, &K) != 2 || L < 0 || K < 1 || L > MAXL) {
        set_err("basis: bad shell header");
        free(buf);
        return -1;
      }
      rec_elem* r = &tab[current];
      r->s = realloc(r->s, sizeof(rec_shell) * (size_t)(r->n + 1));
      rec_shell* sh = &r->s[r->n++];
      sh->L = L;
      sh->K = K;
      sh->e = malloc(sizeof(double) * (size_t)K);
      sh->c = malloc(sizeof(double) * (size_t)K);
      for (int k = 0; k < K; ++k) {
        char* row = next_line(&cur);
        char es[64], cs[64];
        if (!row || sscanf(trim(row), "%63s %63s", es, cs) != 2 || !parse_num(es, &sh->e[k]) ||
            !parse_num(cs, &sh->c[k]) || sh->e[k] <= 0.0) {
          set_err("basis: bad primitive row");
          free(buf);
          return -1;
        }
      }
    }
  }
  free(buf);
  return 0;
}

/* parse_xyz (molecule.hpp:105-158) */
static int parse_xyz(const char* text, orc_ctx* C) {
  char* buf = dup_str(text);
  char* cur = buf;
  char* line = next_line(&cur);
  long declared;
  if (!line || sscanf(trim(line), "%ld", &declared) != 1 || declared < 0) {
    set_err("xyz: bad atom count");
    free(buf);
    return -1;
  }
  if (!next_line(&cur)) {
    set_err("xyz: unexpected end of file");
    free(buf);
    return -1;
  }
  C->Z = malloc(sizeof(int) * (size_t)(declared + 1));
  C->pos = malloc(sizeof(double) * 3 * (size_t)(declared + 1));
  int n = 0;
  while ((line = next_line(&cur))) {
    char* t = trim(line);
    if (!*t) continue;
    char sym[16], xs[64], ys[64], zs[64];
    double x, y, z;
    if (n >= declared || sscanf(t, "%15s %63s %63s %63s", sym, xs, ys, zs) != 4 ||
        !parse_num(xs, &x) || !parse_num(ys, &y) || !parse_num(zs, &z)) {
      set_err("xyz: bad atom line or count mismatch");
      free(buf);
      return -1;
    }
    int Z = atomic_number_of(sym);
    if (!Z) {
      set_err("xyz: unknown element");
      free(buf);
      return -1;
    }
    C->Z[n] = Z;
    /* Vec3(x,y,z) * angstrom_to_bohr: element-wise */
    C->pos[3 * n] = x * ANG2BOHR;
    C->pos[3 * n + 1] = y * ANG2BOHR;
    C->pos[3 * n + 2] = z * ANG2BOHR;
    ++n;
  }
  free(buf);
  if (n != declared) {
    set_err("xyz: declared atom count differs");
    return -1;
  }
  C->natoms = n;
  return 0;
}

/* primitive_pair_overlap / primitive_norm (basis_set.hpp:112-120) */
static double prim_pair_overlap(double a, double b, int L) {
  double p = a + b;
  return pow(M_PI / p, 1.5) * odf(L) / pow(2.0 * p, L);
}

/* attach_basis (basis_set.hpp:127-155) */
static int attach_basis(orc_ctx* C, rec_elem* tab) {
  int ns = 0;
  for (int a = 0; a < C->natoms; ++a) {
    if (!tab[C->Z[a]].n) {
      set_err("basis table lacks an element of the molecule");
      return -1;
    }
    ns += tab[C->Z[a]].n;
  }
  C->nshell = ns;
  C->sh = calloc((size_t)ns, sizeof(shell_t));
  int s = 0;
  for (int a = 0; a < C->natoms; ++a) {
    rec_elem* r = &tab[C->Z[a]];
    for (int k = 0; k < r->n; ++k, ++s) {
      shell_t* sh = &C->sh[s];
      memcpy(sh->c, &C->pos[3 * a], sizeof sh->c);
      sh->L = r->s[k].L;
      sh->K = r->s[k].K;
      sh->atom = a;
      sh->exps = malloc(sizeof(double) * (size_t)sh->K);
      sh->coefs = malloc(sizeof(double) * (size_t)sh->K);
      memcpy(sh->exps, r->s[k].e, sizeof(double) * (size_t)sh->K);
      memcpy(sh->coefs, r->s[k].c, sizeof(double) * (size_t)sh->K);
      for (int q = 0; q < sh->K; ++q)
        sh->coefs[q] *= 1.0 / sqrt(prim_pair_overlap(sh->exps[q], sh->exps[q], sh->L));
      double self = 0.0;
      for (int q = 0; q < sh->K; ++q)
        for (int l = 0; l < sh->K; ++l)
          self += sh->coefs[q] * sh->coefs[l] * prim_pair_overlap(sh->exps[q], sh->exps[l], sh->L);
      const double scale = 1.0 / sqrt(self);
      for (int q = 0; q < sh->K; ++q) sh->coefs[q] *= scale;
    }
  }
  C->bf_off = malloc(sizeof(int) * (size_t)(ns + 1));
  int off = 0;
  for (int q = 0; q < ns; ++q) {
    C->bf_off[q] = off;
    off += ncart(C->sh[q].L);
  }
  C->bf_off[ns] = off;
  C->nbf = off;
  return 0;
}

/* ------------------------------------------------------------ pair store */
static int pair_cmp(const void* a, const void* b) {
  const pair_t* x = a;
  const pair_t* y = b;
  int kx[5] = {x->li + x->lj, x->li, x->lj, x->i, x->j};
  int ky[5] = {y->li + y->lj, y->li, y->lj, y->i, y->j};
  for (int q = 0; q < 5; ++q)
    if (kx[q] != ky[q]) return kx[q] < ky[q] ? -1 : 1;
  return 0;
}

/* build_pairs (block.hpp:52-103) */
static void build_pairs(orc_ctx* C, double thr) {
  const int S = C->nshell;
  C->pr = calloc((size_t)S * (size_t)(S + 1) / 2, sizeof(pair_t));
  int np = 0;
  for (int i = 0; i < S; ++i)
    for (int j = i; j < S; ++j) {
      const shell_t* a = &C->sh[i];
      const shell_t* b = &C->sh[j];
      pair_t* sp = &C->pr[np];
      sp->i = i;
      sp->j = j;
      sp->li = a->L;
      sp->lj = b->L;
      for (int d = 0; d < 3; ++d) sp->AB[d] = a->c[d] - b->c[d];
      const double ab2 = sp->AB[0] * sp->AB[0] + sp->AB[1] * sp->AB[1] + sp->AB[2] * sp->AB[2];
      sp->prims = malloc(sizeof(prim_t) * (size_t)(a->K * b->K));
      sp->nprim = 0;
      for (int k = 0; k < a->K; ++k)
        for (int l = 0; l < b->K; ++l) {
          const double alpha = a->exps[k], beta = b->exps[l];
          prim_t pp;
          pp.p = alpha + beta;
          pp.inv_two_p = 0.5 / pp.p;
          for (int d = 0; d < 3; ++d) {
            pp.P[d] = (alpha * a->c[d] + beta * b->c[d]) / pp.p;
            pp.PA[d] = pp.P[d] - a->c[d];
            pp.PB[d] = pp.P[d] - b->c[d];
          }
          pp.kappa = exp(-alpha * beta * ab2 / pp.p);
          pp.coef = a->coefs[k] * b->coefs[l];
          if (thr > 0.0 && fabs(pp.coef) * pp.kappa < thr) continue;
          sp->prims[sp->nprim++] = pp;
        }
      if (thr > 0.0 && sp->nprim == 0) {
        free(sp->prims);
        continue;
      }
      ++np;
    }
  C->npair = np;
  qsort(C->pr, (size_t)np, sizeof(pair_t), pair_cmp); /* keys unique: stable */
}

/* tile_pairs (block.hpp:115-131) and make_blocks (block.hpp:135-150) */
static void build_tiles(orc_ctx* C, int M) {
  C->tl = malloc(sizeof(tile_t) * (size_t)(C->npair + 1));
  C->ntile = 0;
  int start = 0, n = C->npair;
  while (start < n) {
    int end = start;
    while (end < n && C->pr[end].li == C->pr[start].li && C->pr[end].lj == C->pr[start].lj) ++end;
    for (int t = start; t < end; t += M) {
      tile_t* tt = &C->tl[C->ntile++];
      tt->li = C->pr[start].li;
      tt->lj = C->pr[start].lj;
      tt->first = t;
      tt->count = end - t < M ? end - t : M;
    }
    start = end;
  }
  long long T = C->ntile;
  C->nblock = T * (T + 1) / 2;
  C->bl = malloc(sizeof(block_t) * (size_t)(C->nblock + 1));
  long long b = 0;
  for (int ti = 0; ti < C->ntile; ++ti)
    for (int tj = ti; tj < C->ntile; ++tj) {
      C->bl[b].bt = ti;
      C->bl[b].kt = tj;
      ++b;
    }
}

orc_ctx* orc_create(const char* xyz_text, const char* basis_text, double kappa_screen,
                    int tile_size) {
  pthread_once(&g_once, init_tables);
  if (tile_size < 1) {
    set_err("tile_pairs: tile size must be >= 1");
    return NULL;
  }
  orc_ctx* C = calloc(1, sizeof(orc_ctx));
  rec_elem tab[37];
  memset(tab, 0, sizeof tab);
  int ok = parse_xyz(xyz_text, C) == 0 && parse_basis(basis_text, tab) == 0 &&
           attach_basis(C, tab) == 0;
  for (int z = 0; z < 37; ++z) {
    for (int k = 0; k < tab[z].n; ++k) {
      free(tab[z].s[k].e);
      free(tab[z].s[k].c);
    }
    free(tab[z].s);
  }
  if (!ok) {
    orc_destroy(C);
    return NULL;
  }
  if (C->nshell == 0) {
    set_err("build_pairs: no shells");
    orc_destroy(C);
    return NULL;
  }
  build_pairs(C, kappa_screen);
  build_tiles(C, tile_size);
  return C;
}

void orc_destroy(orc_ctx* C) {
  if (!C) return;
  for (int s = 0; s < C->nshell && C->sh; ++s) {
    free(C->sh[s].exps);
    free(C->sh[s].coefs);
  }
  for (int x = 0; x < C->npair; ++x) free(C->pr[x].prims);
  free(C->sh);
  free(C->pr);
  free(C->tl);
  free(C->bl);
  free(C->bf_off);
  free(C->Z);
  free(C->pos);
  free(C->Q);
  free(C);
}

int orc_nbf(orc_ctx* C) { return C->nbf; }
int orc_nshells(orc_ctx* C) { return C->nshell; }
int orc_npairs(orc_ctx* C) { return C->npair; }
int orc_ntiles(orc_ctx* C) { return C->ntile; }
long long orc_nblocks(orc_ctx* C) { return C->nblock; }
int orc_natoms(orc_ctx* C) { return C->natoms; }
int orc_nelectrons(orc_ctx* C) {
  int n = 0;
  for (int a = 0; a < C->natoms; ++a) n += C->Z[a];
  return n;
}
void orc_atoms(orc_ctx* C, int* Z, double* pos) {
  memcpy(Z, C->Z, sizeof(int) * (size_t)C->natoms);
  memcpy(pos, C->pos, sizeof(double) * 3 * (size_t)C->natoms);
}
void orc_shells(orc_ctx* C, int* L, int* K, int* atom, int* bf_off, double* center) {
  for (int s = 0; s < C->nshell; ++s) {
    L[s] = C->sh[s].L;
    K[s] = C->sh[s].K;
    atom[s] = C->sh[s].atom;
    bf_off[s] = C->bf_off[s];
    memcpy(&center[3 * s], C->sh[s].c, sizeof(double) * 3);
  }
}
void orc_shell_prims(orc_ctx* C, int s, double* exps, double* coefs) {
  memcpy(exps, C->sh[s].exps, sizeof(double) * (size_t)C->sh[s].K);
  memcpy(coefs, C->sh[s].coefs, sizeof(double) * (size_t)C->sh[s].K);
}
void orc_pairs(orc_ctx* C, int* i, int* j, int* nprim) {
  for (int x = 0; x < C->npair; ++x) {
    i[x] = C->pr[x].i;
    j[x] = C->pr[x].j;
    nprim[x] = C->pr[x].nprim;
  }
}
void orc_pair_prims(orc_ctx* C, int x, double* rec) {
  const pair_t* sp = &C->pr[x];
  for (int k = 0; k < sp->nprim; ++k) {
    const prim_t* p = &sp->prims[k];
    double* o = rec + 13 * k;
    o[0] = p->p;
    o[1] = p->inv_two_p;
    for (int d = 0; d < 3; ++d) {
      o[2 + d] = p->P[d];
      o[5 + d] = p->PA[d];
      o[8 + d] = p->PB[d];
    }
    o[11] = p->kappa;
    o[12] = p->coef;
  }
}
void orc_tiles(orc_ctx* C, int* li, int* lj, int* first, int* count) {
  for (int t = 0; t < C->ntile; ++t) {
    li[t] = C->tl[t].li;
    lj[t] = C->tl[t].lj;
    first[t] = C->tl[t].first;
    count[t] = C->tl[t].count;
  }
}

/* ------------------------------------------------------------------ ERI */
typedef struct {
  double* V; /* primitive VRR table [m][e][f] */
  double* Cc; /* contracted [e][f] */
  double* HB; /* bra HRR [b][a][f] */
  double* HK; /* ket HRR [d][c] */
  double* raw;
  size_t capV, capC, capHB, capHK, capRaw;
} scratch_t;

static double* grow(double** p, size_t* cap, size_t n) {
  if (n > *cap) {
    free(*p);
    *p = malloc(sizeof(double) * n);
    *cap = n;
  }
  return *p;
}

/* One shell quartet (bra pair b, ket pair k): raw contracted integrals,
 * a-major over components of (b.i, b.j, k.i, k.j). Binding per SPEC.md:290,
 * 316 and SURVEY.md Appendix C; recurrences per dag.hpp:125-170. */
static int eri_raw(const pair_t* b, const pair_t* k, scratch_t* S) {
  const int la = b->li, lb = b->lj, lc = k->li, ld = k->lj;
  const int Lab = la + lb, Lcd = lc + ld, M = Lab + Lcd;
  const int ne = cart_off(Lab + 1), nf = cart_off(Lcd + 1), nm = M + 1;
  double* V = grow(&S->V, &S->capV, (size_t)nm * ne * nf);
  double* Cc = grow(&S->Cc, &S->capC, (size_t)ne * nf);
  memset(Cc, 0, sizeof(double) * (size_t)ne * nf);
#define VV(m, e, f) V[((size_t)(m) * ne + (e)) * nf + (f)]
  const double two_pi_25 = 2.0 * pow(M_PI, 2.5);
  double F[MAXLT + 1];
  for (int ia = 0; ia < b->nprim; ++ia) {
    const prim_t* a = &b->prims[ia];
    for (int ic = 0; ic < k->nprim; ++ic) {
      const prim_t* c = &k->prims[ic];
      const double pq = a->p + c->p;
      const double rho = a->p * c->p / pq;
      double W[3], WP[3], WQ[3], PQ[3];
      for (int d = 0; d < 3; ++d) {
        W[d] = (a->p * a->P[d] + c->p * c->P[d]) / pq;
        WP[d] = W[d] - a->P[d];
        WQ[d] = W[d] - c->P[d];
        PQ[d] = a->P[d] - c->P[d];
      }
      const double T = rho * (PQ[0] * PQ[0] + PQ[1] * PQ[1] + PQ[2] * PQ[2]);
      const double pref = two_pi_25 / (a->p * c->p * sqrt(pq)) * a->kappa * c->kappa;
      orc_boys(M, T, F);
      const double i2p = a->inv_two_p, i2q = c->inv_two_p, i2pq = 0.5 / pq;
      const double rp = rho / a->p, rq = rho / c->p;
      /* bra vertical relation, f = 0 (dag.hpp:133-140) */
      for (int m = 0; m <= M; ++m) VV(m, 0, 0) = pref * F[m];
      for (int e = 1; e < ne; ++e) {
        const int* em = g_mom[e];
        const int et = em[0] + em[1] + em[2];
        int i = em[0] ? 0 : (em[1] ? 1 : 2);
        int m1[3] = {em[0], em[1], em[2]};
        m1[i] -= 1;
        const int e1 = idx3(m1[0], m1[1], m1[2]);
        int e2 = -1;
        if (m1[i] > 0) {
          int m2[3] = {m1[0], m1[1], m1[2]};
          m2[i] -= 1;
          e2 = idx3(m2[0], m2[1], m2[2]);
        }
        for (int m = 0; m <= M - et; ++m) {
          double v = a->PA[i] * VV(m, e1, 0) + WP[i] * VV(m + 1, e1, 0);
          if (e2 >= 0) v += m1[i] * i2p * (VV(m, e2, 0) - rp * VV(m + 1, e2, 0));
          VV(m, e, 0) = v;
        }
      }
      /* ket vertical relation (dag.hpp:148-163) */
      for (int f = 1; f < nf; ++f) {
        const int* fm = g_mom[f];
        const int ft = fm[0] + fm[1] + fm[2];
        int i = fm[0] ? 0 : (fm[1] ? 1 : 2);
        int n1[3] = {fm[0], fm[1], fm[2]};
        n1[i] -= 1;
        const int f1 = idx3(n1[0], n1[1], n1[2]);
        int f2 = -1;
        if (n1[i] > 0) {
          int n2[3] = {n1[0], n1[1], n1[2]};
          n2[i] -= 1;
          f2 = idx3(n2[0], n2[1], n2[2]);
        }
        for (int e = 0; e < ne; ++e) {
          const int* em = g_mom[e];
          const int et = em[0] + em[1] + em[2];
          int em1 = -1;
          if (em[i] > 0) {
            int q[3] = {em[0], em[1], em[2]};
            q[i] -= 1;
            em1 = idx3(q[0], q[1], q[2]);
          }
          for (int m = 0; m <= M - et - ft; ++m) {
            double v = c->PA[i] * VV(m, e, f1) + WQ[i] * VV(m + 1, e, f1);
            if (f2 >= 0) v += n1[i] * i2q * (VV(m, e, f2) - rq * VV(m + 1, e, f2));
            if (em1 >= 0) v += em[i] * i2pq * VV(m + 1, em1, f1);
            VV(m, e, f) = v;
          }
        }
      }
      /* contraction boundary (compiler.hpp:143) */
      const double w = a->coef * c->coef;
      for (int e = cart_off(la); e < ne; ++e)
        for (int f = cart_off(lc); f < nf; ++f) Cc[(size_t)e * nf + f] += w * VV(0, e, f);
    }
  }
#undef VV
  /* bra horizontal relation on contracted values (dag.hpp:141-147):
   * [a (b+1_i)| = [(a+1_i) b| + AB_i [a b| */
  const int nbm = cart_off(lb + 1);
  double* HB = grow(&S->HB, &S->capHB, (size_t)nbm * ne * nf);
#define H(bb, aa, f) HB[((size_t)(bb) * ne + (aa)) * nf + (f)]
  for (int e = 0; e < ne; ++e)
    for (int f = 0; f < nf; ++f) H(0, e, f) = Cc[(size_t)e * nf + f];
  for (int bt = 1; bt <= lb; ++bt)
    for (int bb = cart_off(bt); bb < cart_off(bt + 1); ++bb) {
      const int* bm = g_mom[bb];
      int i = bm[0] ? 0 : (bm[1] ? 1 : 2);
      int q[3] = {bm[0], bm[1], bm[2]};
      q[i] -= 1;
      const int b1 = idx3(q[0], q[1], q[2]);
      for (int at = la; at <= Lab - bt; ++at)
        for (int aa = cart_off(at); aa < cart_off(at + 1); ++aa) {
          const int* am = g_mom[aa];
          int r[3] = {am[0], am[1], am[2]};
          r[i] += 1;
          const int a1 = idx3(r[0], r[1], r[2]);
          for (int f = 0; f < nf; ++f) H(bb, aa, f) = H(b1, a1, f) + b->AB[i] * H(b1, aa, f);
        }
    }
  /* ket horizontal relation (dag.hpp:164-170), per bra target */
  const int na = ncart(la), nb = ncart(lb), nc = ncart(lc), nd = ncart(ld);
  const int ndm = cart_off(ld + 1);
  double* HK = grow(&S->HK, &S->capHK, (size_t)ndm * nf);
  double* raw = grow(&S->raw, &S->capRaw, (size_t)na * nb * nc * nd);
  size_t n = 0;
  for (int ia = 0; ia < na; ++ia)
    for (int ib = 0; ib < nb; ++ib) {
      const int ag = cart_off(la) + ia, bg = cart_off(lb) + ib;
      for (int f = 0; f < nf; ++f) HK[f] = H(bg, ag, f);
      for (int dt = 1; dt <= ld; ++dt)
        for (int dd = cart_off(dt); dd < cart_off(dt + 1); ++dd) {
          const int* dm = g_mom[dd];
          int i = dm[0] ? 0 : (dm[1] ? 1 : 2);
          int q[3] = {dm[0], dm[1], dm[2]};
          q[i] -= 1;
          const int d1 = idx3(q[0], q[1], q[2]);
          for (int ct = lc; ct <= Lcd - dt; ++ct)
            for (int cc = cart_off(ct); cc < cart_off(ct + 1); ++cc) {
              const int* cm = g_mom[cc];
              int r[3] = {cm[0], cm[1], cm[2]};
              r[i] += 1;
              const int c1 = idx3(r[0], r[1], r[2]);
              HK[(size_t)dd * nf + cc] = HK[(size_t)d1 * nf + c1] + k->AB[i] * HK[(size_t)d1 * nf + cc];
            }
        }
      for (int ic = 0; ic < nc; ++ic)
        for (int id = 0; id < nd; ++id)
          raw[n++] = HK[(size_t)(cart_off(ld) + id) * nf + cart_off(lc) + ic];
    }
#undef H
  return (int)n;
}

/* Scale by prod component_norm_scale (Appendix C), value *= ((sa*sb)*sc)*sd. */
static int eri_scaled(const orc_ctx* C, int x, int y, scratch_t* S, double* out) {
  const pair_t* b = &C->pr[x];
  const pair_t* k = &C->pr[y];
  int n = eri_raw(b, k, S);
  const int ls[4] = {b->li, b->lj, k->li, k->lj};
  double sc[4][ (MAXL + 1) * (MAXL + 2) / 2 ];
  for (int q = 0; q < 4; ++q)
    for (int c = 0; c < ncart(ls[q]); ++c) sc[q][c] = comp_scale(g_mom[cart_off(ls[q]) + c]);
  size_t t = 0;
  for (int a = 0; a < ncart(ls[0]); ++a)
    for (int bb = 0; bb < ncart(ls[1]); ++bb)
      for (int c = 0; c < ncart(ls[2]); ++c)
        for (int d = 0; d < ncart(ls[3]); ++d, ++t)
          out[t] = S->raw[t] * (sc[0][a] * sc[1][bb] * sc[2][c] * sc[3][d]);
  return n;
}

int orc_eri_quartet(orc_ctx* C, int x, int y, double* out) {
  pthread_once(&g_once, init_tables);
  if (x < 0 || y < 0 || x >= C->npair || y >= C->npair) {
    set_err("eri_quartet: pair index out of range");
    return -1;
  }
  scratch_t S;
  memset(&S, 0, sizeof S);
  int n = eri_scaled(C, x, y, &S, out);
  free(S.V);
  free(S.Cc);
  free(S.HB);
  free(S.HK);
  free(S.raw);
  return n;
}

/* ------------------------------------------------------------- threading */
typedef struct {
  orc_ctx* C;
  long long next; /* shared counter (atomic) */
  const double* D;
  double tau;
  long long stride, offset;
  int nthreads;
  double** Jp;
  double** Kp;
  long long* nq;
  int mode; /* 0 = Q, 1 = JK */
  const unsigned char* nzb; /* D-sparse builds: per shell pair (s*nshell+t), D block nonzero */
  const int* lx;            /* explicit quartet list (build_jk_list), else NULL */
  const int* ly;
  long long nlist;
} job_t;

typedef struct {
  job_t* job;
  int w;
} warg_t;

static int keep(const orc_ctx* C, double tau, int x, int y) {
  return tau <= 0.0 || C->Q[x] * C->Q[y] >= tau;
}

static void* q_worker(void* arg) {
  warg_t* wa = arg;
  job_t* J = wa->job;
  orc_ctx* C = J->C;
  scratch_t S;
  memset(&S, 0, sizeof S);
  double out[ (MAXL + 1) * (MAXL + 2) / 2 * (MAXL + 1) * (MAXL + 2) / 2 *
              (MAXL + 1) * (MAXL + 2) / 2 * (MAXL + 1) * (MAXL + 2) / 2 ];
  for (;;) {
    long long x = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
    if (x >= C->npair) break;
    eri_scaled(C, (int)x, (int)x, &S, out);
    const int ni = ncart(C->pr[x].li), nj = ncart(C->pr[x].lj);
    double mx = 0.0;
    for (int m = 0; m < ni; ++m)
      for (int n = 0; n < nj; ++n) {
        double v = fabs(out[(((size_t)m * nj + n) * ni + m) * nj + n]);
        if (v > mx) mx = v;
      }
    C->Q[x] = sqrt(mx);
  }
  free(S.V);
  free(S.Cc);
  free(S.HB);
  free(S.HK);
  free(S.raw);
  return NULL;
}

static int run_workers(job_t* J, void* (*fn)(void*)) {
  int nt = J->nthreads;
  pthread_t* th = malloc(sizeof(pthread_t) * (size_t)nt);
  warg_t* wa = malloc(sizeof(warg_t) * (size_t)nt);
  for (int w = 0; w < nt; ++w) {
    wa[w].job = J;
    wa[w].w = w;
    pthread_create(&th[w], NULL, fn, &wa[w]);
  }
  for (int w = 0; w < nt; ++w) pthread_join(th[w], NULL);
  free(th);
  free(wa);
  return 0;
}

static int default_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static void compute_q(orc_ctx* C) {
  if (C->have_q) return;
  free(C->Q);
  C->Q = calloc((size_t)C->npair, sizeof(double));
  job_t J;
  memset(&J, 0, sizeof J);
  J.C = C;
  J.nthreads = default_threads();
  run_workers(&J, q_worker);
  C->have_q = 1;
}

int orc_schwarz(orc_ctx* C, double* Q) {
  pthread_once(&g_once, init_tables);
  compute_q(C);
  memcpy(Q, C->Q, sizeof(double) * (size_t)C->npair);
  return 0;
}
void orc_set_schwarz(orc_ctx* C, const double* Q) {
  free(C->Q);
  C->Q = malloc(sizeof(double) * (size_t)C->npair);
  memcpy(C->Q, Q, sizeof(double) * (size_t)C->npair);
  C->have_q = 1;
}

long long orc_quartets(orc_ctx* C, double tau, int* xs, int* ys, long long cap) {
  pthread_once(&g_once, init_tables);
  if (tau > 0.0) compute_q(C);
  long long n = 0;
  for (long long bi = 0; bi < C->nblock; ++bi) {
    const tile_t* ti = &C->tl[C->bl[bi].bt];
    const tile_t* tj = &C->tl[C->bl[bi].kt];
    for (int x = ti->first; x < ti->first + ti->count; ++x) {
      int y0 = C->bl[bi].bt == C->bl[bi].kt ? x : tj->first;
      for (int y = y0; y < tj->first + tj->count; ++y)
        if (keep(C, tau, x, y)) {
          if (n < cap) {
            xs[n] = x;
            ys[n] = y;
          }
          ++n;
        }
    }
  }
  return n;
}

/* Digestion of one canonical quartet. */
static void digest(const orc_ctx* C, int x, int y, const double* v, const double* D, double* J,
                   double* K) {
  const pair_t* b = &C->pr[x];
  const pair_t* k = &C->pr[y];
  const int si = b->i, sj = b->j, sk = k->i, sl = k->j;
  const size_t oi = (size_t)C->bf_off[si], oj = (size_t)C->bf_off[sj];
  const size_t ok = (size_t)C->bf_off[sk], ol = (size_t)C->bf_off[sl];
  const int ni = ncart(b->li), nj = ncart(b->lj), nk = ncart(k->li), nl = ncart(k->lj);
  const double deg = (si != sj ? 2.0 : 1.0) * (sk != sl ? 2.0 : 1.0) * (x != y ? 2.0 : 1.0);
  const double q = 0.25 * deg;
  const size_t N = (size_t)C->nbf;
  size_t n = 0;
  for (int m = 0; m < ni; ++m)
    for (int nn = 0; nn < nj; ++nn)
      for (int l = 0; l < nk; ++l)
        for (int s = 0; s < nl; ++s, ++n) {
          const size_t mu = oi + m, nu = oj + nn, la = ok + l, sg = ol + s;
          const double val = v[n];
          J[mu * N + nu] += D[la * N + sg] * val * deg;
          J[la * N + sg] += D[mu * N + nu] * val * deg;
          K[mu * N + la] += q * D[nu * N + sg] * val;
          K[nu * N + sg] += q * D[mu * N + la] * val;
          K[mu * N + sg] += q * D[nu * N + la] * val;
          K[nu * N + la] += q * D[mu * N + sg] * val;
        }
}

/* D-sparse skip (orc_build_jk_dsparse): every one of the six D blocks the
 * quartet reads is zero, so its J/K contributions are exactly zero. */
static int d_blocks_zero(const orc_ctx* C, const unsigned char* nzb, int x, int y) {
  const int S = C->nshell;
  const int i = C->pr[x].i, j = C->pr[x].j, k = C->pr[y].i, l = C->pr[y].j;
  return !(nzb[k * S + l] | nzb[i * S + j] | nzb[j * S + l] | nzb[i * S + k] | nzb[j * S + k] |
           nzb[i * S + l]);
}

static void* jk_worker(void* arg) {
  warg_t* wa = arg;
  job_t* J = wa->job;
  orc_ctx* C = J->C;
  scratch_t S;
  memset(&S, 0, sizeof S);
  double* out = malloc(sizeof(double) * 50625); /* (g g|g g) */
  long long nq = 0;
  for (;;) {
    /* only the sampled blocks offset, offset + stride, ... are claimed */
    const long long st = J->stride > 1 ? J->stride : 1, o0 = J->stride > 1 ? J->offset : 0;
    const long long k = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
    const long long bi = o0 + k * st;
    if (bi >= C->nblock) break;
    const tile_t* ti = &C->tl[C->bl[bi].bt];
    const tile_t* tj = &C->tl[C->bl[bi].kt];
    for (int x = ti->first; x < ti->first + ti->count; ++x) {
      int y0 = C->bl[bi].bt == C->bl[bi].kt ? x : tj->first;
      for (int y = y0; y < tj->first + tj->count; ++y) {
        if (!keep(C, J->tau, x, y)) continue;
        if (J->nzb && d_blocks_zero(C, J->nzb, x, y)) continue;
        eri_scaled(C, x, y, &S, out);
        digest(C, x, y, out, J->D, J->Jp[wa->w], J->Kp[wa->w]);
        ++nq;
      }
    }
  }
  J->nq[wa->w] = nq;
  free(out);
  free(S.V);
  free(S.Cc);
  free(S.HB);
  free(S.HK);
  free(S.raw);
  return NULL;
}

/* Worker over an explicit canonical quartet list (x <= y), 1024 at a time. */
static void* jk_list_worker(void* arg) {
  warg_t* wa = arg;
  job_t* J = wa->job;
  orc_ctx* C = J->C;
  scratch_t S;
  memset(&S, 0, sizeof S);
  double* out = malloc(sizeof(double) * 50625);
  long long nq = 0;
  for (;;) {
    const long long b = 1024 * __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
    if (b >= J->nlist) break;
    const long long e = b + 1024 < J->nlist ? b + 1024 : J->nlist;
    for (long long q = b; q < e; ++q) {
      eri_scaled(C, J->lx[q], J->ly[q], &S, out);
      digest(C, J->lx[q], J->ly[q], out, J->D, J->Jp[wa->w], J->Kp[wa->w]);
      ++nq;
    }
  }
  J->nq[wa->w] = nq;
  free(out);
  free(S.V);
  free(S.Cc);
  free(S.HB);
  free(S.HK);
  free(S.raw);
  return NULL;
}

static int jk_run(orc_ctx* C, const double* D, double tau, int nthreads, long long stride,
                  long long offset, const unsigned char* nzb, const int* lx, const int* ly,
                  long long nlist, double* Jout, double* Kout, long long* nquartets, double* seconds);

int orc_build_jk_timed(orc_ctx* C, const double* D, double tau, int nthreads, long long stride,
                       long long offset, double* Jout, double* Kout, long long* nquartets,
                       double* seconds) {
  return jk_run(C, D, tau, nthreads, stride, offset, NULL, NULL, NULL, 0, Jout, Kout, nquartets, seconds);
}

int orc_build_jk_dsparse(orc_ctx* C, const double* D, double tau, int nthreads, double* Jout,
                         double* Kout, long long* nquartets) {
  pthread_once(&g_once, init_tables);
  const int S = C->nshell;
  const size_t N = (size_t)C->nbf;
  unsigned char* nzb = calloc((size_t)S * (size_t)S, 1);
  for (int s = 0; s < S; ++s)
    for (int t = 0; t < S; ++t) {
      const int ns = ncart(C->sh[s].L), nt = ncart(C->sh[t].L);
      unsigned char nz = 0;
      for (int m = 0; m < ns && !nz; ++m)
        for (int n = 0; n < nt; ++n)
          if (D[(size_t)(C->bf_off[s] + m) * N + (size_t)(C->bf_off[t] + n)] != 0.0) {
            nz = 1;
            break;
          }
      nzb[s * S + t] = nz;
    }
  const int rc = jk_run(C, D, tau, nthreads, 1, 0, nzb, NULL, NULL, 0, Jout, Kout, nquartets, NULL);
  free(nzb);
  return rc;
}

int orc_build_jk_list(orc_ctx* C, const double* D, long long n, const int* xs, const int* ys,
                      int nthreads, double* Jout, double* Kout) {
  for (long long q = 0; q < n; ++q)
    if (xs[q] < 0 || ys[q] < xs[q] || ys[q] >= C->npair) {
      set_err("build_jk_list: quartets must be canonical pair-store indices x <= y < npairs");
      return -1;
    }
  return jk_run(C, D, 0.0, nthreads, 1, 0, NULL, xs, ys, n, Jout, Kout, NULL, NULL);
}

/* Per pair x: canonical survivors (x, y >= x) in block order and the wrapping
 * sum of splitmix64(y) (compact list identity at sizes too large to export). */
typedef struct {
  orc_ctx* C;
  double tau;
  long long next;
  long long** cnt;
  unsigned long long** hs;
} surv_job_t;
typedef struct {
  surv_job_t* job;
  int w;
} surv_arg_t;
static unsigned long long splitmix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static void* surv_worker(void* arg) {
  surv_arg_t* a = arg;
  surv_job_t* J = a->job;
  const orc_ctx* C = J->C;
  long long* cn = J->cnt[a->w];
  unsigned long long* hs = J->hs[a->w];
  for (;;) {
    const long long bi = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
    if (bi >= C->nblock) break;
    const tile_t* ti = &C->tl[C->bl[bi].bt];
    const tile_t* tj = &C->tl[C->bl[bi].kt];
    for (int x = ti->first; x < ti->first + ti->count; ++x) {
      int y0 = C->bl[bi].bt == C->bl[bi].kt ? x : tj->first;
      for (int y = y0; y < tj->first + tj->count; ++y)
        if (keep(C, J->tau, x, y)) {
          ++cn[x];
          hs[x] += splitmix64((unsigned long long)y);
        }
    }
  }
  return NULL;
}
long long orc_pair_survivors(orc_ctx* C, double tau, long long* count, unsigned long long* ysum) {
  pthread_once(&g_once, init_tables);
  if (tau > 0.0) compute_q(C);
  const int nt = default_threads();
  surv_job_t J;
  memset(&J, 0, sizeof J);
  J.C = C;
  J.tau = tau;
  J.cnt = malloc(sizeof(long long*) * (size_t)nt);
  J.hs = malloc(sizeof(unsigned long long*) * (size_t)nt);
  for (int w = 0; w < nt; ++w) {
    J.cnt[w] = calloc((size_t)C->npair, sizeof(long long));
    J.hs[w] = calloc((size_t)C->npair, sizeof(unsigned long long));
  }
  pthread_t* th = malloc(sizeof(pthread_t) * (size_t)nt);
  surv_arg_t* wa = malloc(sizeof(surv_arg_t) * (size_t)nt);
  for (int w = 0; w < nt; ++w) {
    wa[w].job = &J;
    wa[w].w = w;
    pthread_create(&th[w], NULL, surv_worker, &wa[w]);
  }
  for (int w = 0; w < nt; ++w) pthread_join(th[w], NULL);
  long long total = 0;
  for (int x = 0; x < C->npair; ++x) {
    long long c = 0;
    unsigned long long h = 0;
    for (int w = 0; w < nt; ++w) {
      c += J.cnt[w][x];
      h += J.hs[w][x];
    }
    count[x] = c;
    ysum[x] = h;
    total += c;
  }
  for (int w = 0; w < nt; ++w) {
    free(J.cnt[w]);
    free(J.hs[w]);
  }
  free(J.cnt);
  free(J.hs);
  free(th);
  free(wa);
  return total;
}

static int jk_run(orc_ctx* C, const double* D, double tau, int nthreads, long long stride,
                  long long offset, const unsigned char* nzb, const int* lx, const int* ly,
                  long long nlist, double* Jout, double* Kout, long long* nquartets, double* seconds) {
  pthread_once(&g_once, init_tables);
  if (tau > 0.0) compute_q(C);
  if (nthreads <= 0) nthreads = default_threads();
  const size_t N = (size_t)C->nbf, NN = N * N;
  job_t J;
  memset(&J, 0, sizeof J);
  J.C = C;
  J.D = D;
  J.tau = tau;
  J.stride = stride;
  J.offset = offset;
  J.nthreads = nthreads;
  J.nzb = nzb;
  J.lx = lx;
  J.ly = ly;
  J.nlist = nlist;
  J.Jp = malloc(sizeof(double*) * (size_t)nthreads);
  J.Kp = malloc(sizeof(double*) * (size_t)nthreads);
  J.nq = calloc((size_t)nthreads, sizeof(long long));
  for (int w = 0; w < nthreads; ++w) {
    J.Jp[w] = calloc(NN, sizeof(double));
    J.Kp[w] = calloc(NN, sizeof(double));
  }
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  run_workers(&J, lx ? jk_list_worker : jk_worker);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  if (seconds) *seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  double* Jm = calloc(NN, sizeof(double));
  double* Km = calloc(NN, sizeof(double));
  long long nq = 0;
  for (int w = 0; w < nthreads; ++w) {
    for (size_t e = 0; e < NN; ++e) {
      Jm[e] += J.Jp[w][e];
      Km[e] += J.Kp[w][e];
    }
    nq += J.nq[w];
    free(J.Jp[w]);
    free(J.Kp[w]);
  }
  for (size_t a = 0; a < N; ++a)
    for (size_t bb = 0; bb < N; ++bb) {
      Jout[a * N + bb] = 0.25 * (Jm[a * N + bb] + Jm[bb * N + a]);
      Kout[a * N + bb] = 0.5 * (Km[a * N + bb] + Km[bb * N + a]);
    }
  if (nquartets) *nquartets = nq;
  free(Jm);
  free(Km);
  free(J.Jp);
  free(J.Kp);
  free(J.nq);
  return 0;
}

int orc_build_jk_sample(orc_ctx* C, const double* D, double tau, int nthreads, long long stride,
                        long long offset, double* J, double* K, long long* nquartets) {
  return orc_build_jk_timed(C, D, tau, nthreads, stride, offset, J, K, nquartets, NULL);
}

int orc_build_jk(orc_ctx* C, const double* D, double tau, int nthreads, double* J, double* K,
                 long long* nquartets) {
  return orc_build_jk_timed(C, D, tau, nthreads, 1, 0, J, K, nquartets, NULL);
}

/* ------------------------------------------------- one-electron (SPEC §scf) */
/* McMurchie–Davidson Hermite expansion: E[i][j][t] for one dimension. */
static void hermite_E(int la, int lb, double a, double b, double XAB, double* E /* [la+1][lb+3][la+lb+3] */,
                      int sj, int st) {
  const double p = a + b, mu = a * b / p;
  const double XPA = -b / p * XAB, XPB = a / p * XAB;
  const double i2p = 0.5 / p;
#define EE(i, j, t) E[((i) * sj + (j)) * st + (t)]
  for (int i = 0; i <= la; ++i)
    for (int j = 0; j < sj; ++j)
      for (int t = 0; t < st; ++t) EE(i, j, t) = 0.0;
  EE(0, 0, 0) = exp(-mu * XAB * XAB);
  for (int i = 0; i <= la; ++i)
    for (int j = 0; j < sj; ++j) {
      if (i == 0 && j == 0) continue;
      for (int t = 0; t <= i + j && t < st; ++t) {
        double v;
        if (j == 0) {
          v = XPA * EE(i - 1, 0, t) + (t + 1 < st ? (t + 1) * EE(i - 1, 0, t + 1) : 0.0);
          if (t > 0) v += i2p * EE(i - 1, 0, t - 1);
        } else {
          v = XPB * EE(i, j - 1, t) + (t + 1 < st ? (t + 1) * EE(i, j - 1, t + 1) : 0.0);
          if (t > 0) v += i2p * EE(i, j - 1, t - 1);
        }
        EE(i, j, t) = v;
      }
    }
#undef EE
  (void)lb;
}

int orc_one_electron(orc_ctx* C, double* Sm, double* Tm, double* Vm) {
  pthread_once(&g_once, init_tables);
  const size_t N = (size_t)C->nbf;
  memset(Sm, 0, sizeof(double) * N * N);
  memset(Tm, 0, sizeof(double) * N * N);
  memset(Vm, 0, sizeof(double) * N * N);
  enum { LM = MAXL + 1, SJ = MAXL + 3, ST = 2 * MAXL + 4 };
  double E[3][LM * SJ * ST];
  for (int s1 = 0; s1 < C->nshell; ++s1)
    for (int s2 = 0; s2 < C->nshell; ++s2) {
      const shell_t* A = &C->sh[s1];
      const shell_t* B = &C->sh[s2];
      const int na = ncart(A->L), nb = ncart(B->L);
      for (int ka = 0; ka < A->K; ++ka)
        for (int kb = 0; kb < B->K; ++kb) {
          const double a = A->exps[ka], b = B->exps[kb], p = a + b;
          const double w = A->coefs[ka] * B->coefs[kb];
          double P[3];
          for (int d = 0; d < 3; ++d) {
            hermite_E(A->L, B->L + 2, a, b, A->c[d] - B->c[d], E[d], SJ, ST);
            P[d] = (a * A->c[d] + b * B->c[d]) / p;
          }
          const double s3 = pow(M_PI / p, 1.5);
          /* nuclear attraction: Hermite Coulomb integrals R_tuv per nucleus */
          const int Lt = A->L + B->L;
          for (int ia = 0; ia < na; ++ia)
            for (int ib = 0; ib < nb; ++ib) {
              const int* ma = g_mom[cart_off(A->L) + ia];
              const int* mb = g_mom[cart_off(B->L) + ib];
              double s1d[3], t1d[3];
              for (int d = 0; d < 3; ++d) {
                const double* Ed = E[d];
                const int i = ma[d], j = mb[d];
#define EE(i, j, t) Ed[((i) * SJ + (j)) * ST + (t)]
                s1d[d] = EE(i, j, 0);
                double t = 4.0 * b * b * EE(i, j + 2, 0) - 2.0 * b * (2 * j + 1) * EE(i, j, 0);
                if (j >= 2) t += (double)(j * (j - 1)) * EE(i, j - 2, 0);
                t1d[d] = t;
#undef EE
              }
              const size_t mu = (size_t)C->bf_off[s1] + ia, nu = (size_t)C->bf_off[s2] + ib;
              Sm[mu * N + nu] += w * s3 * s1d[0] * s1d[1] * s1d[2];
              Tm[mu * N + nu] += w * s3 * -0.5 *
                                 (t1d[0] * s1d[1] * s1d[2] + s1d[0] * t1d[1] * s1d[2] +
                                  s1d[0] * s1d[1] * t1d[2]);
            }
          for (int at = 0; at < C->natoms; ++at) {
            double PC[3];
            for (int d = 0; d < 3; ++d) PC[d] = P[d] - C->pos[3 * at + d];
            const double RPC2 = PC[0] * PC[0] + PC[1] * PC[1] + PC[2] * PC[2];
            double F[2 * MAXL + 1];
            orc_boys(Lt, p * RPC2, F);
            /* R[n][t][u][v] */
            enum { R1 = 2 * MAXL + 1 };
            static __thread double R[R1][R1][R1][R1];
            for (int n = 0; n <= Lt; ++n) R[n][0][0][0] = pow(-2.0 * p, n) * F[n];
            for (int n = Lt - 1; n >= 0; --n) {
              const int rem = Lt - n;
              for (int t = 0; t <= rem; ++t)
                for (int u = 0; u <= rem - t; ++u)
                  for (int v = 0; v <= rem - t - u; ++v) {
                    if (t + u + v == 0) continue;
                    double val;
                    if (t > 0) {
                      val = PC[0] * R[n + 1][t - 1][u][v];
                      if (t > 1) val += (t - 1) * R[n + 1][t - 2][u][v];
                    } else if (u > 0) {
                      val = PC[1] * R[n + 1][t][u - 1][v];
                      if (u > 1) val += (u - 1) * R[n + 1][t][u - 2][v];
                    } else {
                      val = PC[2] * R[n + 1][t][u][v - 1];
                      if (v > 1) val += (v - 1) * R[n + 1][t][u][v - 2];
                    }
                    R[n][t][u][v] = val;
                  }
            }
            const double pre = -C->Z[at] * 2.0 * M_PI / p * w;
            for (int ia = 0; ia < na; ++ia)
              for (int ib = 0; ib < nb; ++ib) {
                const int* ma = g_mom[cart_off(A->L) + ia];
                const int* mb = g_mom[cart_off(B->L) + ib];
                double s = 0.0;
                for (int t = 0; t <= ma[0] + mb[0]; ++t)
                  for (int u = 0; u <= ma[1] + mb[1]; ++u)
                    for (int v = 0; v <= ma[2] + mb[2]; ++v)
                      s += E[0][(ma[0] * SJ + mb[0]) * ST + t] * E[1][(ma[1] * SJ + mb[1]) * ST + u] *
                           E[2][(ma[2] * SJ + mb[2]) * ST + v] * R[0][t][u][v];
                const size_t mu = (size_t)C->bf_off[s1] + ia, nu = (size_t)C->bf_off[s2] + ib;
                Vm[mu * N + nu] += pre * s;
              }
          }
        }
    }
  /* component normalisation (molecule.hpp:207-213) */
  double* sc = malloc(sizeof(double) * N);
  for (int s = 0; s < C->nshell; ++s)
    for (int c = 0; c < ncart(C->sh[s].L); ++c)
      sc[C->bf_off[s] + c] = comp_scale(g_mom[cart_off(C->sh[s].L) + c]);
  for (size_t a = 0; a < N; ++a)
    for (size_t b = 0; b < N; ++b) {
      const double f = sc[a] * sc[b];
      Sm[a * N + b] *= f;
      Tm[a * N + b] *= f;
      Vm[a * N + b] *= f;
    }
  free(sc);
  return 0;
}

double orc_nuclear_repulsion(orc_ctx* C) {
  double e = 0.0;
  for (int a = 0; a < C->natoms; ++a)
    for (int b = a + 1; b < C->natoms; ++b) {
      double d2 = 0.0;
      for (int k = 0; k < 3; ++k) {
        double d = C->pos[3 * a + k] - C->pos[3 * b + k];
        d2 += d * d;
      }
      e += (double)C->Z[a] * C->Z[b] / sqrt(d2);
    }
  return e;
}
