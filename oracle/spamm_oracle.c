/*
 * spamm_oracle.c — plain, slow, obviously-correct CPU oracle of the SpAMM
 * product and the dual-channel Newton-Schulz iteration of
 *   Challacombe, Haut & Bock, "A N-Body Solver for Square Root Iteration"
 *   (arXiv 1508.05856, PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1508_05856_b200/csrc) and never calls it.
 *
 * Everything is IEEE fp64, round-to-nearest-even, compiled WITHOUT fp
 * contraction and without fast-math (reading L19), with a pointer
 * quadtree exactly as PAPER.md describes it:
 *
 *   quadtree a^i, children a^{i+1}_{00,01,10,11}
 *   ||a^i||_F = sqrt(sum_children ||a^{i+1}_xy||_F^2)
 *   Eq. newspamm, with the canonical 2x2 block product in
 *   place of the misprinted quadrants (reading L1):
 *     a (x)_tau b = 0                    if ||a|| ||b|| < tau ||A|| ||B||
 *                 = a . b                if leaf (N_b x N_b dense product)
 *                 = [a00(x)b00 + a01(x)b10 ,  a00(x)b01 + a01(x)b11 ;
 *                    a10(x)b00 + a11(x)b10 ,  a10(x)b01 + a11(x)b11 ]
 *   ||A||, ||B|| are the root norms of this call's operands.
 *   An absent sub-block (zero marker, norm 0) contributes nothing and is not
 *   a leaf task, at any tau including 0 (reading L3/L6).
 *
 *   Dual NS iteration in north_star form (BJ:5, Eq. cannonical P:383-389,
 *   reading L8):  X = Z (x)_tau Y;  t_k = (n - tr X)/n;
 *   H = 1/2 (3I - X) (h_alpha at alpha = 1);  Y <- Y (x)_tau_s H;
 *   Z <- H (x)_tau Z.  Y0 = s/c, Z0 = I, c ~ ||s||_2.
 *
 * Parity pins: see tests/test_oracle_pins.py and DESIGN.md §4.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct onode {
    double norm;           /* Frobenius norm (not squared)   */
    struct onode *ch[4];   /* 00, 01, 10, 11; NULL = zero marker        */
    double *blk;           /* leaf only: N_b x N_b row-major            */
} onode;

typedef struct omat {
    int n, b, nb, L;       /* n = b * 2^L */
    onode *root;
} omat;

/* ---------------------------------------------------------------- tasks */
typedef struct {
    int32_t *ikj;          /* 3 * cap */
    int64_t cap, count;
    int record;
} taskrec;

static void rec_task(taskrec *r, int i, int k, int j)
{
    if (!r || !r->record) return;
#pragma omp critical(oracle_tasks)
    {
        if (r->count < r->cap) {
            r->ikj[3 * r->count + 0] = i;
            r->ikj[3 * r->count + 1] = k;
            r->ikj[3 * r->count + 2] = j;
        }
        r->count++;
    }
}

/* ------------------------------------------------------------ node utils */
static onode *new_interior(void)
{
    onode *p = (onode *)calloc(1, sizeof(onode));
    return p;
}

static onode *new_leaf(int b)
{
    onode *p = (onode *)calloc(1, sizeof(onode));
    p->blk = (double *)malloc(sizeof(double) * (size_t)b * b);
    return p;
}

static void free_node(onode *p)
{
    if (!p) return;
    for (int c = 0; c < 4; c++) free_node(p->ch[c]);
    free(p->blk);
    free(p);
}

/* Leaf norm: sqrt of the row-major sum of squares (P:125-129 at the leaf). */
static double leaf_norm(const double *x, int b)
{
    double s = 0.0;
    for (int r = 0; r < b * b; r++) s += x[r] * x[r];
    return sqrt(s);
}

/* Interior norm from the four children, in order 00,01,10,11. */
static double interior_norm(const onode *p)
{
    double s = 0.0;
    for (int c = 0; c < 4; c++)
        if (p->ch[c]) s += p->ch[c]->norm * p->ch[c]->norm;
    return sqrt(s);
}

/* Finalise a leaf: an all-zero block is a zero marker (reading L6). */
static onode *finish_leaf(onode *p, int b)
{
    p->norm = leaf_norm(p->blk, b);
    if (p->norm == 0.0) { free_node(p); return NULL; }
    return p;
}

/* Finalise an interior node: decorations in backward recursion. */
static onode *finish_interior(onode *p)
{
    if (!p->ch[0] && !p->ch[1] && !p->ch[2] && !p->ch[3]) { free(p); return NULL; }
    p->norm = interior_norm(p);
    return p;
}

/* --------------------------------------------------------------- build */
/* dense: n x n row-major (ld = n).  Sub-block (i0, j0) of side w. */
static onode *build_rec(const double *dense, int n, int b, int i0, int j0, int w)
{
    if (w == b) {
        onode *p = new_leaf(b);
        for (int r = 0; r < b; r++)
            memcpy(p->blk + (size_t)r * b, dense + (size_t)(i0 + r) * n + j0,
                   sizeof(double) * b);
        return finish_leaf(p, b);
    }
    int h = w / 2;
    onode *p = new_interior();
    p->ch[0] = build_rec(dense, n, b, i0, j0, h);
    p->ch[1] = build_rec(dense, n, b, i0, j0 + h, h);
    p->ch[2] = build_rec(dense, n, b, i0 + h, j0, h);
    p->ch[3] = build_rec(dense, n, b, i0 + h, j0 + h, h);
    return finish_interior(p);
}

static int ilog2(int v) { int l = 0; while ((1 << l) < v) l++; return l; }

omat *or_build(const double *dense, int n, int b)
{
    if (b < 1 || n < b || n % b) return NULL;
    int nb = n / b;
    if ((nb & (nb - 1)) != 0) return NULL;
    omat *m = (omat *)calloc(1, sizeof(omat));
    m->n = n; m->b = b; m->nb = nb; m->L = ilog2(nb);
    m->root = build_rec(dense, n, b, 0, 0, n);
    return m;
}

/* Insert a leaf block at block coordinates (I, J) (descending from the root). */
static void insert_leaf(omat *m, int I, int J, const double *blk)
{
    onode **pp = &m->root;
    for (int lev = 0; lev < m->L; lev++) {
        if (!*pp) *pp = new_interior();
        int sh = m->L - 1 - lev;
        int c = (((I >> sh) & 1) << 1) | ((J >> sh) & 1);
        pp = &(*pp)->ch[c];
    }
    if (!*pp) *pp = new_leaf(m->b);
    memcpy((*pp)->blk, blk, sizeof(double) * (size_t)m->b * m->b);
}

/* Recompute all norms bottom-up, dropping zero blocks (reading L6). */
static onode *renorm(onode *p, int lev, int L, int b)
{
    if (!p) return NULL;
    if (lev == L) return finish_leaf(p, b);
    for (int c = 0; c < 4; c++) p->ch[c] = renorm(p->ch[c], lev + 1, L, b);
    return finish_interior(p);
}

omat *or_build_blocks(int n, int b, int64_t nblk, const int32_t *bi,
                      const int32_t *bj, const double *blocks)
{
    if (b < 1 || n < b || n % b) return NULL;
    int nb = n / b;
    if ((nb & (nb - 1)) != 0) return NULL;
    omat *m = (omat *)calloc(1, sizeof(omat));
    m->n = n; m->b = b; m->nb = nb; m->L = ilog2(nb);
    for (int64_t t = 0; t < nblk; t++)
        insert_leaf(m, bi[t], bj[t], blocks + (size_t)t * b * b);
    m->root = renorm(m->root, 0, m->L, b);
    return m;
}

void or_free(omat *m)
{
    if (!m) return;
    free_node(m->root);
    free(m);
}

double or_norm(const omat *m) { return m->root ? m->root->norm : 0.0; }
int or_n(const omat *m) { return m->n; }
int or_b(const omat *m) { return m->b; }

static void to_dense_rec(const onode *p, int n, int b, int i0, int j0, int w, double *out)
{
    if (!p) return;
    if (w == b) {
        for (int r = 0; r < b; r++)
            memcpy(out + (size_t)(i0 + r) * n + j0, p->blk + (size_t)r * b,
                   sizeof(double) * b);
        return;
    }
    int h = w / 2;
    to_dense_rec(p->ch[0], n, b, i0, j0, h, out);
    to_dense_rec(p->ch[1], n, b, i0, j0 + h, h, out);
    to_dense_rec(p->ch[2], n, b, i0 + h, j0, h, out);
    to_dense_rec(p->ch[3], n, b, i0 + h, j0 + h, h, out);
}

void or_to_dense(const omat *m, double *out)
{
    memset(out, 0, sizeof(double) * (size_t)m->n * m->n);
    to_dense_rec(m->root, m->n, m->b, 0, 0, m->n, out);
}

/* Node norms of one level (0 = root, L = leaves), row-major 2^lev x 2^lev. */
static void level_norms_rec(const onode *p, int lev, int target, int I, int J,
                            int side, double *out)
{
    if (!p) return;
    if (lev == target) { out[(size_t)I * side + J] = p->norm; return; }
    for (int c = 0; c < 4; c++)
        level_norms_rec(p->ch[c], lev + 1, target, 2 * I + (c >> 1), 2 * J + (c & 1),
                        side, out);
}

void or_level_norms(const omat *m, int level, double *out)
{
    int side = 1 << level;
    memset(out, 0, sizeof(double) * (size_t)side * side);
    level_norms_rec(m->root, 0, level, 0, 0, side, out);
}

static const onode *find_leaf(const omat *m, int I, int J)
{
    const onode *p = m->root;
    for (int lev = 0; lev < m->L && p; lev++) {
        int sh = m->L - 1 - lev;
        p = p->ch[(((I >> sh) & 1) << 1) | ((J >> sh) & 1)];
    }
    return p;
}

/* Copy block (I,J) into out; returns 1 if present, 0 if absent (zeros). */
int or_get_block(const omat *m, int I, int J, double *out)
{
    const onode *p = find_leaf(m, I, J);
    if (!p) { memset(out, 0, sizeof(double) * (size_t)m->b * m->b); return 0; }
    memcpy(out, p->blk, sizeof(double) * (size_t)m->b * m->b);
    return 1;
}

static int64_t count_rec(const onode *p, int lev, int L)
{
    if (!p) return 0;
    if (lev == L) return 1;
    int64_t s = 0;
    for (int c = 0; c < 4; c++) s += count_rec(p->ch[c], lev + 1, L);
    return s;
}

int64_t or_nblocks(const omat *m) { return count_rec(m->root, 0, m->L); }

/* Present blocks, in row-major (I,J) order. */
int64_t or_block_coords(const omat *m, int32_t *bi, int32_t *bj, int64_t cap)
{
    int64_t c = 0;
    for (int I = 0; I < m->nb; I++)
        for (int J = 0; J < m->nb; J++)
            if (find_leaf(m, I, J)) {
                if (c < cap) { bi[c] = I; bj[c] = J; }
                c++;
            }
    return c;
}

/* ------------------------------------------------------------- SpAMM */
typedef struct {
    int b, L;
    double thr;          /* tau * ||A|| * ||B|| */
    taskrec *rec;
    int par_depth;       /* spawn OpenMP tasks above this depth */
} mulctx;

/* p + q (elementwise on the quadtree), consuming both. */
static onode *add_consume(onode *p, onode *q, int lev, int L, int b)
{
    if (!p) return q;
    if (!q) return p;
    if (lev == L) {
        for (int r = 0; r < b * b; r++) p->blk[r] = p->blk[r] + q->blk[r];
        free_node(q);
        return finish_leaf(p, b);
    }
    for (int c = 0; c < 4; c++) {
        p->ch[c] = add_consume(p->ch[c], q->ch[c], lev + 1, L, b);
        q->ch[c] = NULL;
    }
    free_node(q);
    return finish_interior(p);
}

/* Leaf product c = a . b, plain triple loop, k ascending. */
static onode *leaf_product(const double *a, const double *bb, int b)
{
    onode *p = new_leaf(b);
    double *c = p->blk;
    for (int i = 0; i < b; i++) {
        for (int j = 0; j < b; j++) c[(size_t)i * b + j] = 0.0;
        for (int k = 0; k < b; k++) {
            double aik = a[(size_t)i * b + k];
            for (int j = 0; j < b; j++)
                c[(size_t)i * b + j] = c[(size_t)i * b + j] + aik * bb[(size_t)k * b + j];
        }
    }
    return finish_leaf(p, b);
}

/* Eq. newspamm.  (i,k,j): block coordinates at depth lev. */
static onode *spamm_rec(const onode *a, const onode *b, int lev, int i, int k, int j,
                        const mulctx *cx)
{
    if (!a || !b) return NULL;                         /* zero marker          */
    if (a->norm * b->norm < cx->thr) return NULL;      /* occlusion cull P:205 */
    if (lev == cx->L) {                                /* leaf: dense product  */
        rec_task(cx->rec, i, k, j);
        return leaf_product(a->blk, b->blk, cx->b);
    }
    onode *c = new_interior();
    onode *t[4][2];
    /* c_xy = a_x0 (x) b_0y + a_x1 (x) b_1y   (canonical 2x2, reading L1) */
    if (lev < cx->par_depth) {
        for (int x = 0; x < 2; x++)
            for (int y = 0; y < 2; y++)
                for (int z = 0; z < 2; z++) {
#pragma omp task shared(t) firstprivate(x, y, z)
                    t[2 * x + y][z] = spamm_rec(a->ch[2 * x + z], b->ch[2 * z + y], lev + 1,
                                                2 * i + x, 2 * k + z, 2 * j + y, cx);
                }
#pragma omp taskwait
    } else {
        for (int x = 0; x < 2; x++)
            for (int y = 0; y < 2; y++)
                for (int z = 0; z < 2; z++)
                    t[2 * x + y][z] = spamm_rec(a->ch[2 * x + z], b->ch[2 * z + y], lev + 1,
                                                2 * i + x, 2 * k + z, 2 * j + y, cx);
    }
    for (int q = 0; q < 4; q++)
        c->ch[q] = add_consume(t[q][0], t[q][1], lev + 1, cx->L, cx->b);
    return finish_interior(c);
}

/* C = A (x)_tau B.  tasks (nullable): recorded leaf triples (i,k,j), up to cap;
 * *ntasks receives the full count.  Returns NULL on shape mismatch / tau < 0. */
omat *or_multiply(const omat *A, const omat *B, double tau, int32_t *tasks,
                  int64_t cap, int64_t *ntasks)
{
    if (!A || !B || A->n != B->n || A->b != B->b) return NULL;
    if (!(tau >= 0.0)) return NULL;
    taskrec rec = { tasks, cap, 0, tasks != NULL || ntasks != NULL };
    mulctx cx;
    cx.b = A->b; cx.L = A->L;
    cx.thr = tau * or_norm(A) * or_norm(B);
    cx.rec = &rec;
    cx.par_depth = 3;
    omat *C = (omat *)calloc(1, sizeof(omat));
    C->n = A->n; C->b = A->b; C->nb = A->nb; C->L = A->L;
#pragma omp parallel
#pragma omp single
    C->root = spamm_rec(A->root, B->root, 0, 0, 0, 0, &cx);
    if (ntasks) *ntasks = rec.count;
    return C;
}

/* ------------------------------------------------------ elementwise maps */
static onode *copy_node(const onode *p, int lev, int L, int b)
{
    if (!p) return NULL;
    if (lev == L) {
        onode *q = new_leaf(b);
        memcpy(q->blk, p->blk, sizeof(double) * (size_t)b * b);
        q->norm = p->norm;
        return q;
    }
    onode *q = new_interior();
    for (int c = 0; c < 4; c++) q->ch[c] = copy_node(p->ch[c], lev + 1, L, b);
    q->norm = p->norm;
    return q;
}

/* Transpose: children 01 <-> 10, leaves transposed; every node keeps its norm
 * (the Frobenius norm is transpose-invariant: ||a^T|| = ||a||, so a^T's
 * decorations are a's, bitwise). */
static onode *transpose_node(const onode *p, int lev, int L, int b)
{
    if (!p) return NULL;
    if (lev == L) {
        onode *q = new_leaf(b);
        for (int r = 0; r < b; r++)
            for (int c = 0; c < b; c++) q->blk[(size_t)c * b + r] = p->blk[(size_t)r * b + c];
        q->norm = p->norm;
        return q;
    }
    onode *q = new_interior();
    q->ch[0] = transpose_node(p->ch[0], lev + 1, L, b);
    q->ch[1] = transpose_node(p->ch[2], lev + 1, L, b);
    q->ch[2] = transpose_node(p->ch[1], lev + 1, L, b);
    q->ch[3] = transpose_node(p->ch[3], lev + 1, L, b);
    q->norm = p->norm;
    return q;
}

omat *or_transpose(const omat *m)
{
    omat *c = (omat *)calloc(1, sizeof(omat));
    *c = *m;
    c->root = transpose_node(m->root, 0, m->L, m->b);
    return c;
}

/* A^T (x)_tau B: the SpAMM product (Eq. newspamm) of the transposed quadtree. */
omat *or_multiply_t(const omat *A, const omat *B, double tau, int32_t *tasks, int64_t cap, int64_t *ntasks)
{
    omat *At = or_transpose(A);
    omat *C = or_multiply(At, B, tau, tasks, cap, ntasks);
    or_free(At);
    return C;
}

omat *or_copy(const omat *m)
{
    omat *c = (omat *)calloc(1, sizeof(omat));
    *c = *m;
    c->root = copy_node(m->root, 0, m->L, m->b);
    return c;
}

/* op 0: y = x / c ;  op 1: y = (x / c + mu*delta) / (1 + mu) ;
 * op 2: y = x * c  ;  op 3: y = x / c  (same as 0; kept for clarity)
 * op 4: H = 1/2 (3 delta - x)  written as 1.5*delta - 0.5*x (exactly equal, the
 *       1/2 scale is exact).  Diagonal blocks absent from x become 1.5 I.
 * op 8: y = x / c + mu delta   (shifted normalised s, regularised slices)
 * op 6: scaled + stabilised map with alpha = c, eps = mu:
 *       x~ = (1 - 2 eps) x + eps delta   ([0,1] -> [eps, 1-eps], "prior to the logistic")
 *       H  = h_alpha[x~] = sqrt(alpha)/2 (3 delta - alpha x~). */
static onode *map_rec(const onode *p, int lev, int L, int b, int I, int J, int op,
                      double c, double mu)
{
    int diag = (I == J);
    int fill = (op == 1 || op == 4 || op == 5 || op == 6 || op == 8);   /* ops that create absent diagonal blocks */
    if (!p && !(diag && fill)) return NULL;
    if (!p && lev < L && diag && fill) {
        onode *q = new_interior();
        for (int ch = 0; ch < 4; ch++)
            q->ch[ch] = map_rec(NULL, lev + 1, L, b, 2 * I + (ch >> 1), 2 * J + (ch & 1),
                                op, c, mu);
        return finish_interior(q);
    }
    if (lev == L) {
        onode *q = new_leaf(b);
        for (int r = 0; r < b; r++)
            for (int s = 0; s < b; s++) {
                double x = p ? p->blk[(size_t)r * b + s] : 0.0;
                double d = (diag && r == s) ? 1.0 : 0.0;
                double y;
                switch (op) {
                case 0: case 3: y = x / c; break;
                case 1: y = (x / c + mu * d) / (1.0 + mu); break;
                case 2: y = x * c; break;
                case 5: y = d; break;
                case 6: {
                    double xt = (1.0 - 2.0 * mu) * x + mu * d;
                    y = (sqrt(c) / 2.0) * (3.0 * d - c * xt);
                    break;
                }
                case 8: y = x / c + mu * d; break;
                default: y = 1.5 * d - 0.5 * x; break;
                }
                q->blk[(size_t)r * b + s] = y;
            }
        return finish_leaf(q, b);
    }
    onode *q = new_interior();
    for (int ch = 0; ch < 4; ch++)
        q->ch[ch] = map_rec(p->ch[ch], lev + 1, L, b, 2 * I + (ch >> 1), 2 * J + (ch & 1),
                            op, c, mu);
    return finish_interior(q);
}

static omat *map_mat(const omat *m, int op, double c, double mu)
{
    omat *r = (omat *)calloc(1, sizeof(omat));
    r->n = m->n; r->b = m->b; r->nb = m->nb; r->L = m->L;
    r->root = map_rec(m->root, 0, m->L, m->b, 0, 0, op, c, mu);
    return r;
}

omat *or_identity(int n, int b)
{
    omat z = { n, b, n / b, ilog2(n / b), NULL };
    return map_mat(&z, 5, 0.0, 0.0);
}

omat *or_scale(const omat *m, double c, int divide)
{
    return map_mat(m, divide ? 0 : 2, c, 0.0);
}

/* Trace: sum of the diagonal entries, strictly ascending row order. */
double or_trace(const omat *m)
{
    double s = 0.0;
    int b = m->b;
    for (int I = 0; I < m->nb; I++) {
        const onode *p = find_leaf(m, I, I);
        if (!p) continue;
        for (int r = 0; r < b; r++) s += p->blk[(size_t)r * b + r];
    }
    return s;
}

/* ---------------------------------------------------- power iteration */
static void spmv_rec(const onode *p, int lev, int L, int b, int I, int J,
                     const double *v, double *w)
{
    if (!p) return;
    if (lev == L) {
        for (int r = 0; r < b; r++) {
            double s = w[(size_t)I * b + r];
            for (int c = 0; c < b; c++) s = s + p->blk[(size_t)r * b + c] * v[(size_t)J * b + c];
            w[(size_t)I * b + r] = s;
        }
        return;
    }
    for (int c = 0; c < 4; c++)
        spmv_rec(p->ch[c], lev + 1, L, b, 2 * I + (c >> 1), 2 * J + (c & 1), v, w);
}

/* c ~ ||s||_2: K power steps from v0 = 1/sqrt(n) * ones, then the Rayleigh
 * quotient v^T s v (reading L12, "easily obtained largest eigenvalue"). */
double or_power_scale(const omat *s, int K)
{
    int n = s->n;
    double *v = (double *)malloc(sizeof(double) * n);
    double *w = (double *)malloc(sizeof(double) * n);
    for (int i = 0; i < n; i++) v[i] = 1.0 / sqrt((double)n);
    for (int it = 0; it < K; it++) {
        memset(w, 0, sizeof(double) * n);
        spmv_rec(s->root, 0, s->L, s->b, 0, 0, v, w);
        double nn = 0.0;
        for (int i = 0; i < n; i++) nn += w[i] * w[i];
        nn = sqrt(nn);
        for (int i = 0; i < n; i++) v[i] = w[i] / nn;
    }
    memset(w, 0, sizeof(double) * n);
    spmv_rec(s->root, 0, s->L, s->b, 0, 0, v, w);
    double c = 0.0;
    for (int i = 0; i < n; i++) c += v[i] * w[i];
    free(v); free(w);
    return c;
}

/* ------------------------------------------------------ Newton-Schulz */
/* One dual step (north_star form, BJ:5):
 *   X = Z (x)_tau Y ; t = (n - tr X)/n ; H = 1/2(3I - X) ;
 *   Y' = Y (x)_tau_s H ; Z' = H (x)_tau Z.
 * counts (nullable): leaf tasks of the 3 products [X, Y', Z'].
 * Returns 0, or -1 on a non-finite t / norm. */
/* The paper's damping sigmoids, functions of the trace error t_k:
 *   alpha(t) = 1 + 1.85 (1 + e^{-50 (t - .35)})^{-1},
 *   eps(t)   = .1 (1 + e^{-75 (t - .30)})^{-1}. */
double or_alpha(double t) { return 1.0 + 1.85 * (1.0 / (1.0 + exp(-50.0 * (t - 0.35)))); }
double or_eps(double t) { return 0.1 * (1.0 / (1.0 + exp(-75.0 * (t - 0.30)))); }

/* map 0: H = 1/2 (3I - X) (alpha = 1, eps = 0: the north_star form);
 * map 1: H = h_alpha[(1 - 2 eps) X + eps I] with alpha(t_k), eps(t_k). */
/* tasks (nullable): the leaf triples (i,k,j) of the three products [X, Y', Z'],
 * tasks[p] holding up to cap triples (counts[] always receives the full counts) */
int or_ns_step_tasks(const omat *Y, const omat *Z, double tau, double tau_s, int map,
                     omat **Yn, omat **Zn, omat **Hout, double *t, int64_t counts[3],
                     int32_t *tX, int32_t *tY, int32_t *tZ, int64_t cap)
{
    int64_t c0 = 0, c1 = 0, c2 = 0;
    omat *X = or_multiply(Z, Y, tau, tX, tX ? cap : 0, &c0);
    double tr = or_trace(X);
    *t = ((double)X->n - tr) / (double)X->n;
    omat *H = map ? map_mat(X, 6, or_alpha(*t), or_eps(*t)) : map_mat(X, 4, 0.0, 0.0);
    or_free(X);
    *Yn = or_multiply(Y, H, tau_s, tY, tY ? cap : 0, &c1);
    *Zn = or_multiply(H, Z, tau, tZ, tZ ? cap : 0, &c2);
    if (counts) { counts[0] = c0; counts[1] = c1; counts[2] = c2; }
    if (Hout) *Hout = H; else or_free(H);
    if (!isfinite(*t) || !isfinite(or_norm(*Yn)) || !isfinite(or_norm(*Zn))) return -1;
    return 0;
}

int or_ns_step_map(const omat *Y, const omat *Z, double tau, double tau_s, int map,
                   omat **Yn, omat **Zn, omat **Hout, double *t, int64_t counts[3])
{
    return or_ns_step_tasks(Y, Z, tau, tau_s, map, Yn, Zn, Hout, t, counts, NULL, NULL, NULL, 0);
}

int or_ns_step(const omat *Y, const omat *Z, double tau, double tau_s,
               omat **Yn, omat **Zn, omat **Hout, double *t, int64_t counts[3])
{
    return or_ns_step_map(Y, Z, tau, tau_s, 0, Yn, Zn, Hout, t, counts);
}

/* Y0 = s/c (mu = 0) or (s/c + mu I)/(1+mu) (reading L13); Z0 = I. */
omat *or_ns_y0(const omat *s, double c, double mu)
{
    if (mu != 0.0) return map_mat(s, 1, c, mu);
    return map_mat(s, 0, c, 0.0);
}

/* Full run: scale > 0 is used as c, else c = or_power_scale(s, power_iters).
 * On return *Yout ~ (s + c mu I)^{1/2}, *Zout ~ (s + c mu I)^{-1/2}
 * (unscaled by sqrt(c (1+mu))).  t_hist [iters], counts [3*iters] nullable.
 * Returns 0 or -1 (non-finite; Y/Z hold the last finite iterates). */
int or_ns_sqrt(const omat *s, double tau, double tau_s, int iters, double scale,
               int power_iters, double mu, double t_stop, int map, omat **Yout, omat **Zout,
               double *t_hist, int64_t *counts, double *c_used, int *iters_done)
{
    double c = scale > 0.0 ? scale : or_power_scale(s, power_iters);
    if (c_used) *c_used = c;
    omat *Y = or_ns_y0(s, c, mu);
    omat *Z = or_identity(s->n, s->b);
    int rc = 0;
    if (iters_done) *iters_done = 0;
    for (int k = 0; k < iters; k++) {
        omat *Yn, *Zn;
        double t;
        rc = or_ns_step_map(Y, Z, tau, tau_s, map, &Yn, &Zn, NULL, &t, counts ? counts + 3 * k : NULL);
        if (t_hist) t_hist[k] = t;
        if (rc) { or_free(Yn); or_free(Zn); break; }
        or_free(Y); or_free(Z);
        Y = Yn; Z = Zn;
        if (iters_done) *iters_done = k + 1;
        /* convergence monitored by the relative trace error */
        if (t_stop > 0.0 && fabs(t) <= t_stop) break;
    }
    double f = sqrt(c * (1.0 + mu));
    *Yout = map_mat(Y, 2, f, 0.0);
    *Zout = map_mat(Z, 0, f, 0.0);
    or_free(Y); or_free(Z);
    return rc;
}

int or_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------- single channel
 * z_k <- z_{k-1} . h[x_{k-1}],  x_k <- z_k^T . s . z_k, with SpAMM products and the
 * sensitive product rightmost:
 *   Z_{k+1} = Z_k (x)_tau H_k,  W = s (x)_tau_s Z_{k+1},  X_{k+1} = Z_{k+1}^T (x)_tau W,
 * t_k = (n - tr X_k)/n, H_k = h(X_k) (map 0: 1/2 (3I - X); map 1: scaled/stabilised).
 * Start Z_0 = I, X_0 = s/c (= Z_0^T s Z_0; reading L11 analogue: s/c is exact here).
 * Output Z -> (s/c)^{-1/2} / sqrt(c) = s^{-1/2};  Y = W * sqrt(c) -> s^{1/2}.
 * counts [3*iters]: tasks of (Z H, s Z, Z^T W). */
int or_ns_sqrt_single(const omat *s, double tau, double tau_s, int iters, double scale, int power_iters,
                      double t_stop, int map, omat **Yout, omat **Zout, double *t_hist, int64_t *counts,
                      double *c_used, int *iters_done)
{
    double c = scale > 0.0 ? scale : or_power_scale(s, power_iters);
    if (c_used) *c_used = c;
    omat *S1 = or_ns_y0(s, c, 0.0);
    omat *Z = or_identity(s->n, s->b);
    omat *X = or_copy(S1);
    omat *W = or_copy(S1);
    int rc = 0;
    if (iters_done) *iters_done = 0;
    for (int k = 0; k < iters; k++) {
        double tr = or_trace(X);
        double t = ((double)X->n - tr) / (double)X->n;
        if (t_hist) t_hist[k] = t;
        omat *H = map ? map_mat(X, 6, or_alpha(t), or_eps(t)) : map_mat(X, 4, 0.0, 0.0);
        int64_t c0 = 0, c1 = 0, c2 = 0;
        omat *Zn = or_multiply(Z, H, tau, NULL, 0, &c0);
        omat *Wn = or_multiply(S1, Zn, tau_s, NULL, 0, &c1);
        omat *Xn = or_multiply_t(Zn, Wn, tau, NULL, 0, &c2);
        if (counts) { counts[3 * k] = c0; counts[3 * k + 1] = c1; counts[3 * k + 2] = c2; }
        or_free(H);
        if (!isfinite(t) || !isfinite(or_norm(Zn)) || !isfinite(or_norm(Xn))) {
            or_free(Zn); or_free(Wn); or_free(Xn);
            rc = -1;
            break;
        }
        or_free(Z); or_free(W); or_free(X);
        Z = Zn; W = Wn; X = Xn;
        if (iters_done) *iters_done = k + 1;
        if (t_stop > 0.0 && fabs(t) <= t_stop) break;
    }
    double f = sqrt(c);
    *Yout = map_mat(W, 2, f, 0.0);
    *Zout = map_mat(Z, 0, f, 0.0);
    or_free(Z); or_free(W); or_free(X); or_free(S1);
    return rc;
}

/* ------------------------------------------ regularised product representation
 * Eq. product_rep (reading L21): slices of shifted, preconditioned
 * residuals, each solved by the dual iteration at the slice precision tau0, chained
 * by products at tau1:
 *   c = ||s||_2 ;  S_i = s/c + mu_i I  (mu_0 > mu_1 > ... , relative shifts)
 *   R_0 = S_0,  R_i = F^T (x)_tau1 (S_i (x)_tau1 F)  (i >= 1)
 *   Z_i = R_i^{-1/2} (dual NS, tau = tau_s = tau0, own scale by power iteration)
 *   F = Z_0,  F <- F (x)_tau1 Z_i
 * Output G = F / sqrt(c): G^T (s + c mu_m I) G ~ I (an inverse factor). */
int or_regularized_factor(const omat *s, double tau0, double tau1, const double *mu, int nslices, int iters,
                          double t_stop, double scale, int power_iters, omat **Gout, double *c_used,
                          int64_t *slice_iters)
{
    double c = scale > 0.0 ? scale : or_power_scale(s, power_iters);
    if (c_used) *c_used = c;
    omat *F = NULL;
    int rc = 0;
    for (int i = 0; i < nslices && !rc; i++) {
        omat *Si = map_mat(s, 8, c, mu[i]);
        omat *R;
        if (!F) {
            R = Si;
        } else {
            omat *W = or_multiply(Si, F, tau1, NULL, 0, NULL);
            R = or_multiply_t(F, W, tau1, NULL, 0, NULL);
            or_free(W);
            or_free(Si);
        }
        omat *Y, *Z;
        int done = 0;
        rc = or_ns_sqrt(R, tau0, tau0, iters, 0.0, power_iters, 0.0, t_stop, 0, &Y, &Z, NULL, NULL, NULL, &done);
        if (slice_iters) slice_iters[i] = done;
        or_free(R);
        or_free(Y);
        if (!F) {
            F = Z;
        } else {
            omat *Fn = or_multiply(F, Z, tau1, NULL, 0, NULL);
            or_free(F);
            or_free(Z);
            F = Fn;
        }
    }
    *Gout = map_mat(F, 0, sqrt(c), 0.0);
    or_free(F);
    return rc;
}
