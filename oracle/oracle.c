/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the complex
 * Winograd F(4x4,3x3) int8 convolution with integer filter-precision scaling
 * (Meng & Brothers, "Efficient Winograd Convolution via Integer Arithmetic",
 * arXiv 1901.01965).  Citations "P:n" are lines of /root/reference/PAPER.md.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path in
 * paper_1901_01965_b200/; the transform matrices below are typed in from the
 * paper independently of the kernels.
 *
 * Every computation is the textbook definition, done with 64-bit integers:
 *   - direct correlation (O1)
 *   - D = B^T d B on the full 6x6 grid, complex
 *   - W = G_int g G_int^T, G_int = 4 G, complex
 *   - per-(cout, position) scale factor n/2^p, steps (a)-(d)
 *     (read per DESIGN.md A3: n = x >> (y-3), p = 10 - y)
 *   - W' = rha(W n / 2^p)                                  P:312, A7
 *   - inverse factor m/2^q, 8-bit m, q in [4,7]            P:366, A8
 *   - M = sum_ci W' (.) D  (schoolbook complex products)
 *   - M'' = rha(M m / 2^q)
 *   - Y = A^T M'' A, full complex product, assert Im Y == 0
 *   - out32 = rha(Re Y / 16)                               P:366, A11
 *   - y8 = clamp(rha(out32 * M0 / 2^S), -128, 127)         DESIGN.md A14
 * The rational F(2x2,3x3) pipeline of P:259-306 follows at the end.
 * No Karatsuba, conjugate shortcut, blocking or fusion is used here: those
 * are the GPU path's optimisations and are checked against this file.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { int64_t re, im; } gint;

/* ---- transform matrices, typed verbatim from the paper -------------------
 * B^T, entries {0, +-1, +-i}; stored as (re, im).            */
static const int BT_RE[6][6] = {
    {1, 0, 0, 0, -1, 0},
    {0, 1, 1, 1, 1, 0},
    {0, -1, 1, -1, 1, 0},
    {0, 0, -1, 0, 1, 0},
    {0, 0, -1, 0, 1, 0},
    {0, -1, 0, 0, 0, 1}};
static const int BT_IM[6][6] = {
    {0, 0, 0, 0, 0, 0},
    {0, 0, 0, 0, 0, 0},
    {0, 0, 0, 0, 0, 0},
    {0, -1, 0, 1, 0, 0},
    {0, 1, 0, -1, 0, 0},
    {0, 0, 0, 0, 0, 0}};
/* G scaled by 4 element-wise (A2): rows
 * (4,0,0) (1,1,1) (1,-1,1) (1,i,-1) (1,-i,-1) (0,0,4).                   */
static const int G4_RE[6][3] = {
    {4, 0, 0}, {1, 1, 1}, {1, -1, 1}, {1, 0, -1}, {1, 0, -1}, {0, 0, 4}};
static const int G4_IM[6][3] = {
    {0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 0}};
/* A^T.                                                       */
static const int AT_RE[4][6] = {
    {1, 1, 1, 1, 1, 0},
    {0, 1, -1, 0, 0, 0},
    {0, 1, 1, -1, -1, 0},
    {0, 1, -1, 0, 0, 1}};
static const int AT_IM[4][6] = {
    {0, 0, 0, 0, 0, 0},
    {0, 0, 0, 1, -1, 0},
    {0, 0, 0, 0, 0, 0},
    {0, 0, 0, -1, 1, 0}};

/* Output divisor: (G_int = 4 G)  =>  Y = 16 * correlation (A2). */
#define OUT_DIV_SHIFT 4

static inline gint gmul(gint a, gint b) { /* schoolbook complex product */
    gint r;
    r.re = a.re * b.re - a.im * b.im;
    r.im = a.re * b.im + a.im * b.re;
    return r;
}
static inline gint gadd(gint a, gint b) { gint r = {a.re + b.re, a.im + b.im}; return r; }

/* round-half-away-from-zero of v / 2^k, k >= 0. */
int64_t oracle_rha_shift(int64_t v, int k) {
    if (k <= 0) return v;
    int64_t a = v < 0 ? -v : v;
    int64_t r = (a + ((int64_t)1 << (k - 1))) >> k;
    return v < 0 ? -r : r;
}

/* Scale factor for a position whose max magnitude is mx, read
 * per DESIGN.md A3: x = floor(target*128/mx); y = floor(log2 x);
 * n = floor(x / 2^(y-3)); p = 10 - y.  Returns 0 and sets n=p=0 when
 * mx <= target ("no scaling").  Returns -1 if p would leave [4,7]. */
int oracle_scale_factor(int64_t mx, int target, int *n, int *p) {
    *n = 0; *p = 0;
    if (mx <= target) return 0;
    /* the paper's 128; the int8-native target (f3, A29) takes one more bit, 256 with
     * p = 11 - y, so that x keeps 4 significant bits down to factor 8/256 (exactly the largest
     * n/2^p <= target/mx, pinned by brute force)                                              */
    const int f3 = target < 255;
    int64_t x = ((int64_t)target * (f3 ? 256 : 128)) / mx;
    if (x <= 0) return -1;
    int y = 0;
    while (((int64_t)1 << (y + 1)) <= x) y++;
    int nn, pp = (f3 ? 11 : 10) - y;
    if (y >= 3) nn = (int)(x >> (y - 3)); else nn = (int)(x << (3 - y));
    /* p in [4,7] for the paper's target 255; the int8-native target (f3, A29) reaches p = 8 */
    if (pp < 4 || pp > (target < 255 ? 8 : 7)) return -1;
    *n = nn; *p = pp;
    return 0;
}

/* 6-bit code (A4): (n << 2) | (p - 4); 0 = unscaled.   */
int oracle_encode_code(int n, int p) { return n == 0 ? 0 : ((n << 2) | (p - 4)); }
/* 7-bit code of the int8-native target (f3, A29): (n << 3) | (p - 4), p in [4,8]. */
int oracle_encode_code7(int n, int p) { return n == 0 ? 0 : ((n << 3) | (p - 4)); }
void oracle_decode_code7(int code, int *n, int *p) {
    if (code == 0) { *n = 0; *p = 0; return; }
    *n = code >> 3; *p = (code & 7) + 4;
}
void oracle_decode_code(int code, int *n, int *p) {
    if (code == 0) { *n = 0; *p = 0; return; }
    *n = code >> 2; *p = (code & 3) + 4;
}

/* Inverse factor (A8/A27): the largest q in {7,...,3} with
 * m = rha(2^(q+p) / n) <= 255.  q = 3 is needed only by n/2^p = 8/128, which
 * int9 weights (uint8 - zero point, f2) reach and int8 weights never do.
 * Returns -1 if none exists.                                             */
int oracle_reverse_factor(int n, int p, int *m, int *q) {
    for (int qq = 7; qq >= 3; qq--) {
        int64_t num = (int64_t)1 << (qq + p);
        /* rha(num / n) for positive num, n: floor((2 num + n) / (2 n)) */
        int64_t mm = (2 * num + n) / (2 * (int64_t)n);
        if (mm <= 255) { *m = (int)mm; *q = qq; return 0; }
    }
    return -1;
}

/* ---- layouts --------------------------------------------------------------
 * layout 0 = NCHW (x [N][C][H][W], w [Cout][Cin][3][3], y [N][Cout][Ho][Wo])
 * layout 1 = NHWC (x [N][H][W][C], w [Cout][3][3][Cin], y [N][Ho][Wo][Cout]) */
/* Element accessors on int16 tensors: the int8 entry points below widen their
 * inputs, the uint8 ones (f2) store x - zx and w - zw (int9).        */
static inline int64_t x_at(const int16_t *x, int layout, int N, int C, int H, int W,
                           int n, int c, int h, int w) {
    (void)N;
    if (h < 0 || h >= H || w < 0 || w >= W) return 0;   /* zero padding */
    if (layout == 0) return x[(((int64_t)n * C + c) * H + h) * W + w];
    return x[(((int64_t)n * H + h) * W + w) * C + c];
}
static inline int64_t w_at(const int16_t *w, int layout, int Cout, int Cin,
                           int co, int ci, int u, int v) {
    (void)Cout;
    if (layout == 0) return w[(((int64_t)co * Cin + ci) * 3 + u) * 3 + v];
    return w[(((int64_t)co * 3 + u) * 3 + v) * Cin + ci];
}
static inline int64_t y_index(int layout, int Cout, int Ho, int Wo, int n, int co, int oy, int ox) {
    if (layout == 0) return (((int64_t)n * Cout + co) * Ho + oy) * Wo + ox;
    return (((int64_t)n * Ho + oy) * Wo + ox) * Cout + co;
}

/* O1: direct correlation, int64 accumulation (A1, A12). */
void oracle_direct_conv16(const int16_t *x, const int16_t *w, int N, int H, int W,
                          int Cin, int Cout, int pad, int layout, int64_t *out) {
    int Ho = H + 2 * pad - 2, Wo = W + 2 * pad - 2;
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int n = 0; n < N; n++)
        for (int co = 0; co < Cout; co++)
            for (int oy = 0; oy < Ho; oy++)
                for (int ox = 0; ox < Wo; ox++) {
                    int64_t acc = 0;
                    for (int ci = 0; ci < Cin; ci++)
                        for (int u = 0; u < 3; u++)
                            for (int v = 0; v < 3; v++)
                                acc += x_at(x, layout, N, Cin, H, W, n, ci, oy + u - pad, ox + v - pad) *
                                       w_at(w, layout, Cout, Cin, co, ci, u, v);
                    out[y_index(layout, Cout, Ho, Wo, n, co, oy, ox)] = acc;
                }
}

/* O3: W = G_int g G_int^T for one 3x3 filter, full 6x6 complex. */
void oracle_filter_tile(const int64_t g[3][3], gint W[6][6]) {
    gint Gg[6][3];
    for (int i = 0; i < 6; i++)
        for (int j = 0; j < 3; j++) {
            gint s = {0, 0};
            for (int k = 0; k < 3; k++) {
                gint a = {G4_RE[i][k], G4_IM[i][k]}, b = {g[k][j], 0};
                s = gadd(s, gmul(a, b));
            }
            Gg[i][j] = s;
        }
    for (int i = 0; i < 6; i++)
        for (int j = 0; j < 6; j++) {
            gint s = {0, 0};
            for (int k = 0; k < 3; k++) {
                gint gt = {G4_RE[j][k], G4_IM[j][k]};   /* (G^T)[k][j] = G[j][k], no conjugation */
                s = gadd(s, gmul(Gg[i][k], gt));
            }
            W[i][j] = s;
        }
}

/* O2: D = B^T d B for one 6x6 patch, full complex. */
void oracle_input_tile(const int64_t d[6][6], gint D[6][6]) {
    gint Bd[6][6];
    for (int i = 0; i < 6; i++)
        for (int j = 0; j < 6; j++) {
            gint s = {0, 0};
            for (int k = 0; k < 6; k++) {
                gint a = {BT_RE[i][k], BT_IM[i][k]}, b = {d[k][j], 0};
                s = gadd(s, gmul(a, b));
            }
            Bd[i][j] = s;
        }
    for (int i = 0; i < 6; i++)
        for (int j = 0; j < 6; j++) {
            gint s = {0, 0};
            for (int k = 0; k < 6; k++) {
                gint b = {BT_RE[j][k], BT_IM[j][k]};    /* B[k][j] = B^T[j][k] */
                s = gadd(s, gmul(Bd[i][k], b));
            }
            D[i][j] = s;
        }
}

/* O9: Y = A^T M A (complex); returns 0 if Im Y == 0 everywhere. */
int oracle_output_tile(const gint M[6][6], int64_t Y[4][4]) {
    gint AM[4][6];
    int ok = 0;
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 6; j++) {
            gint s = {0, 0};
            for (int k = 0; k < 6; k++) {
                gint a = {AT_RE[i][k], AT_IM[i][k]};
                s = gadd(s, gmul(a, M[k][j]));
            }
            AM[i][j] = s;
        }
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) {
            gint s = {0, 0};
            for (int k = 0; k < 6; k++) {
                gint a = {AT_RE[j][k], AT_IM[j][k]};    /* A[k][j] = A^T[j][k] */
                s = gadd(s, gmul(AM[i][k], a));
            }
            if (s.im != 0) ok = -1;
            Y[i][j] = s.re;
        }
    return ok;
}

/* position (r, c) of the 6x6 grid involves +-i (rows/columns 3, 4) */
static inline int Wt_is_complex_pos(int pos) {
    int r = pos / 6, c = pos % 6;
    return r == 3 || r == 4 || c == 3 || c == 4;
}
static inline int64_t max_abs_component(gint v) {
    int64_t a = v.re < 0 ? -v.re : v.re, b = v.im < 0 ? -v.im : v.im;
    return a > b ? a : b;   /* DESIGN.md A5 */
}

/* Offline filter path for a whole layer.
 *   W_out     [Cout][Cin][36][2]  unscaled G_int g G_int^T (may be NULL)
 *   Wp_out    [Cout][Cin][36][2]  W' (scaled where the code != 0)
 *   codes_out [Cout][36]          6-bit codes, 0 = unscaled
 * scaling == 0: every code is 0 and W' = W.   Returns 0, or -1 if a
 * factor falls outside p in [4,7] (cannot happen for int8 weights).       */
int oracle_filter_transform16(const int16_t *w, int Cout, int Cin, int layout, int scaling,
                              int target, int64_t *W_out, int64_t *Wp_out, uint8_t *codes_out) {
    int status = 0;
    gint *Wt = (gint *)malloc(sizeof(gint) * 36 * (size_t)(Cin > 0 ? Cin : 1));
    for (int co = 0; co < Cout; co++) {
        /* step 1: transform all weights for the current OFM */
        for (int ci = 0; ci < Cin; ci++) {
            int64_t g[3][3];
            for (int u = 0; u < 3; u++)
                for (int v = 0; v < 3; v++) g[u][v] = w_at(w, layout, Cout, Cin, co, ci, u, v);
            gint Wt6[6][6];
            oracle_filter_tile(g, Wt6);
            for (int pos = 0; pos < 36; pos++) Wt[(size_t)ci * 36 + pos] = Wt6[pos / 6][pos % 6];
        }
        for (int pos = 0; pos < 36; pos++) {
            /* int8-native target (f3, A29): complex positions bound |Re| + |Im| by 126 so that
             * after rounding Re', Im' and Re' + Im' all fit s8; real positions bound |W| by 127.   */
            const int f3 = target == 127;
            const int is_cpx = Wt_is_complex_pos(pos);
            const int tgt = f3 && is_cpx ? 126 : target;
            /* step 2: max magnitude at this X-Y location across channels */
            int64_t mx = 0;
            for (int ci = 0; ci < Cin; ci++) {
                gint v = Wt[(size_t)ci * 36 + pos];
                int64_t m = f3 ? (v.re < 0 ? -v.re : v.re) + (v.im < 0 ? -v.im : v.im)
                               : max_abs_component(v);
                if (m > mx) mx = m;
            }
            int n = 0, p = 0;
            if (scaling) {      /* steps 3-4 */
                if (oracle_scale_factor(mx, tgt, &n, &p) != 0) { status = -1; n = 0; p = 0; }
            }
            codes_out[(size_t)co * 36 + pos] = (uint8_t)(f3 ? oracle_encode_code7(n, p) : oracle_encode_code(n, p));
            for (int ci = 0; ci < Cin; ci++) {
                gint v = Wt[(size_t)ci * 36 + pos];
                size_t o = (((size_t)co * Cin + ci) * 36 + pos) * 2;
                if (W_out) { W_out[o] = v.re; W_out[o + 1] = v.im; }
                if (n) {          /* downscale W' = rha(W n / 2^p) on re and im */
                    Wp_out[o] = oracle_rha_shift(v.re * n, p);
                    Wp_out[o + 1] = oracle_rha_shift(v.im * n, p);
                } else {
                    Wp_out[o] = v.re; Wp_out[o + 1] = v.im;
                }
            }
        }
    }
    free(Wt);
    return status;
}

/* Input transform of every tile (O1, O2).  D_out [T][Cin][36][2], T = N*th*tw,
 * tile t = (n*th + ty)*tw + tx with patch origin (4ty - pad, 4tx - pad).   */
void oracle_input_transform16(const int16_t *x, int N, int H, int W, int Cin, int pad,
                              int layout, int64_t *D_out) {
    int Ho = H + 2 * pad - 2, Wo = W + 2 * pad - 2;
    int th = (Ho + 3) / 4, tw = (Wo + 3) / 4;
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; n++)
        for (int ty = 0; ty < th; ty++)
            for (int tx = 0; tx < tw; tx++)
                for (int ci = 0; ci < Cin; ci++) {
                    int64_t d[6][6];
                    for (int a = 0; a < 6; a++)
                        for (int b = 0; b < 6; b++)
                            d[a][b] = x_at(x, layout, N, Cin, H, W, n, ci, 4 * ty - pad + a, 4 * tx - pad + b);
                    gint D[6][6];
                    oracle_input_tile(d, D);
                    size_t t = ((size_t)n * th + ty) * tw + tx;
                    for (int pos = 0; pos < 36; pos++) {
                        size_t o = ((t * Cin + ci) * 36 + pos) * 2;
                        D_out[o] = D[pos / 6][pos % 6].re;
                        D_out[o + 1] = D[pos / 6][pos % 6].im;
                    }
                }
}

/* The complete pipeline of the paper (O1-O12).
 *   out32  [y layout] int32 = rha(Re Y / 16), cropped to Ho x Wo
 *   y8     [y layout] int8  = clamp(rha(out32 * M0 / 2^S))  (may be NULL)
 *   M_out  [T][Cout][36][2] M before reverse scaling  (may be NULL)
 *   Mpp_out[T][Cout][36][2] M'' after reverse scaling (may be NULL)
 * Returns 0; -1 on a scale-factor range error; -2 if Im Y != 0 anywhere;
 * -3 if scaling is off and 16 does not divide Y; -4 if |M''| or |Y| would
 * leave int32 (the GPU stores int32, A23).                     */
int oracle_wino_conv16(const int16_t *x, const int16_t *w, int N, int H, int W, int Cin, int Cout,
                       int pad, int layout, int scaling, int target, int32_t M0, int S,
                       int32_t *out32, int8_t *y8, int64_t *M_out, int64_t *Mpp_out) {
    int Ho = H + 2 * pad - 2, Wo = W + 2 * pad - 2;
    int th = (Ho + 3) / 4, tw = (Wo + 3) / 4;
    size_t T = (size_t)N * th * tw;
    int status = 0;
    int64_t *Wp = (int64_t *)malloc(sizeof(int64_t) * 72 * (size_t)Cout * (Cin > 0 ? Cin : 1));
    uint8_t *codes = (uint8_t *)malloc((size_t)Cout * 36);
    int64_t *D = (int64_t *)malloc(sizeof(int64_t) * 72 * T * (Cin > 0 ? Cin : 1));
    if (oracle_filter_transform16(w, Cout, Cin, layout, scaling, target, NULL, Wp, codes) != 0) status = -1;
    oracle_input_transform16(x, N, H, W, Cin, pad, layout, D);
    int bad_im = 0, bad_div = 0, bad_range = 0;
#pragma omp parallel for collapse(2) schedule(dynamic) reduction(| : bad_im, bad_div, bad_range)
    for (long long t = 0; t < (long long)T; t++)
        for (int co = 0; co < Cout; co++) {
            gint M[6][6];
            memset(M, 0, sizeof(M));
            /* Hadamard products accumulated over all channels */
            for (int ci = 0; ci < Cin; ci++)
                for (int pos = 0; pos < 36; pos++) {
                    size_t ow = (((size_t)co * Cin + ci) * 36 + pos) * 2;
                    size_t od = (((size_t)t * Cin + ci) * 36 + pos) * 2;
                    gint a = {Wp[ow], Wp[ow + 1]}, b = {D[od], D[od + 1]};
                    M[pos / 6][pos % 6] = gadd(M[pos / 6][pos % 6], gmul(a, b));
                }
            /* reverse scaling before the final transforms */
            gint Mpp[6][6];
            for (int pos = 0; pos < 36; pos++) {
                gint v = M[pos / 6][pos % 6];
                int n, p, m = 0, q = 0;
                if (target == 127) oracle_decode_code7(codes[(size_t)co * 36 + pos], &n, &p);
                else oracle_decode_code(codes[(size_t)co * 36 + pos], &n, &p);
                if (n) {
                    oracle_reverse_factor(n, p, &m, &q);
                    v.re = oracle_rha_shift(v.re * m, q);
                    v.im = oracle_rha_shift(v.im * m, q);
                }
                Mpp[pos / 6][pos % 6] = v;
                if (v.re > INT32_MAX || v.re < INT32_MIN || v.im > INT32_MAX || v.im < INT32_MIN) bad_range = 1;
                if (M_out) {
                    size_t o = (((size_t)t * Cout + co) * 36 + pos) * 2;
                    M_out[o] = M[pos / 6][pos % 6].re; M_out[o + 1] = M[pos / 6][pos % 6].im;
                }
                if (Mpp_out) {
                    size_t o = (((size_t)t * Cout + co) * 36 + pos) * 2;
                    Mpp_out[o] = v.re; Mpp_out[o + 1] = v.im;
                }
            }
            int64_t Y[4][4];
            if (oracle_output_tile((const gint(*)[6])Mpp, Y) != 0) bad_im = 1;
            int n_img = (int)(t / ((size_t)th * tw));
            int rem = (int)(t % ((size_t)th * tw));
            int ty = rem / tw, tx = rem % tw;
            for (int i = 0; i < 4; i++)
                for (int j = 0; j < 4; j++) {
                    if (Y[i][j] > INT32_MAX || Y[i][j] < INT32_MIN) bad_range = 1;
                    if (!scaling && (Y[i][j] % 16) != 0) bad_div = 1;
                    int oy = 4 * ty + i, ox = 4 * tx + j;
                    if (oy >= Ho || ox >= Wo) continue;          /* crop (O11) */
                    int64_t o32 = oracle_rha_shift(Y[i][j], OUT_DIV_SHIFT);
                    int64_t yi = y_index(layout, Cout, Ho, Wo, n_img, co, oy, ox);
                    out32[yi] = (int32_t)o32;
                    if (y8) {
                        int64_t r = oracle_rha_shift(o32 * (int64_t)M0, S);
                        if (r > 127) r = 127;
                        if (r < -128) r = -128;
                        y8[yi] = (int8_t)r;
                    }
                }
        }
    if (bad_range) status = status ? status : -4;
    if (bad_div) status = status ? status : -3;
    if (bad_im) status = status ? status : -2;
    free(Wp); free(codes); free(D);
    return status;
}

/* ==========================================================================
 * Rational F(2x2,3x3): the configuration the paper evaluates
 * end to end, with the same filter precision scaling.
 *   G' = 2G, typed from P:261-268.
 *   B^T and A^T are the standard F(2,3) matrices of the cited Lavin algorithm
 *   (the paper prints only G', A25); pinned by the closed form
 *   A^T[(G'gG'^T) (.) (B^T d B)]A = 4 * correlation.
 *   Output divisor 4 ("shift right by 1 after each final transform"),
 *   applied as one final rha(Y / 4) (A26).
 * Positions: the 4x4 grid row-major, all 16 real.                          */
static const int G2[4][3] = {{2, 0, 0}, {1, 1, 1}, {1, -1, 1}, {0, 0, 2}};
static const int BT2[4][4] = {{1, 0, -1, 0}, {0, 1, 1, 0}, {0, -1, 1, 0}, {0, 1, 0, -1}};
static const int AT2[2][4] = {{1, 1, 1, 0}, {0, 1, -1, -1}};
#define OUT2_DIV_SHIFT 2

/* W = G' g G'^T. */
void oracle_filter_tile2(const int64_t g[3][3], int64_t W[4][4]) {
    int64_t Gg[4][3];
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 3; j++) {
            int64_t s = 0;
            for (int k = 0; k < 3; k++) s += G2[i][k] * g[k][j];
            Gg[i][j] = s;
        }
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) {
            int64_t s = 0;
            for (int k = 0; k < 3; k++) s += Gg[i][k] * G2[j][k];
            W[i][j] = s;
        }
}
/* D = B^T d B for one 4x4 patch. */
void oracle_input_tile2(const int64_t d[4][4], int64_t D[4][4]) {
    int64_t Bd[4][4];
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) {
            int64_t s = 0;
            for (int k = 0; k < 4; k++) s += BT2[i][k] * d[k][j];
            Bd[i][j] = s;
        }
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) {
            int64_t s = 0;
            for (int k = 0; k < 4; k++) s += Bd[i][k] * BT2[j][k];
            D[i][j] = s;
        }
}
/* Y = A^T M A (2x2). */
void oracle_output_tile2(const int64_t M[4][4], int64_t Y[2][2]) {
    int64_t AM[2][4];
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 4; j++) {
            int64_t s = 0;
            for (int k = 0; k < 4; k++) s += AT2[i][k] * M[k][j];
            AM[i][j] = s;
        }
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 2; j++) {
            int64_t s = 0;
            for (int k = 0; k < 4; k++) s += AM[i][k] * AT2[j][k];
            Y[i][j] = s;
        }
}
void oracle_filter_tile2_64(const int64_t *g9, int64_t *W16) { oracle_filter_tile2((const int64_t(*)[3])g9, (int64_t(*)[4])W16); }
void oracle_input_tile2_64(const int64_t *d16, int64_t *D16) { oracle_input_tile2((const int64_t(*)[4])d16, (int64_t(*)[4])D16); }
void oracle_output_tile2_64(const int64_t *M16, int64_t *Y4) { oracle_output_tile2((const int64_t(*)[4])M16, (int64_t(*)[2])Y4); }

/* Offline F(2x2) filter path (P:317-330 with 16 positions):
 *   W_out [Cout][Cin][16] (may be NULL), Wp_out [Cout][Cin][16], codes_out [Cout][16]. */
int oracle_filter_transform2_16(const int16_t *w, int Cout, int Cin, int layout, int scaling, int target,
                                int64_t *W_out, int64_t *Wp_out, uint8_t *codes_out) {
    int status = 0;
    int64_t *Wt = (int64_t *)malloc(sizeof(int64_t) * 16 * (size_t)(Cin > 0 ? Cin : 1));
    for (int co = 0; co < Cout; co++) {
        for (int ci = 0; ci < Cin; ci++) {          /* step 1: transform all weights of the OFM */
            int64_t g[3][3], W4[4][4];
            for (int u = 0; u < 3; u++)
                for (int v = 0; v < 3; v++) g[u][v] = w_at(w, layout, Cout, Cin, co, ci, u, v);
            oracle_filter_tile2(g, W4);
            for (int pos = 0; pos < 16; pos++) Wt[(size_t)ci * 16 + pos] = W4[pos / 4][pos % 4];
        }
        for (int pos = 0; pos < 16; pos++) {
            int64_t mx = 0;                          /* step 2: max magnitude across channels */
            for (int ci = 0; ci < Cin; ci++) {
                int64_t v = Wt[(size_t)ci * 16 + pos];
                if (v < 0) v = -v;
                if (v > mx) mx = v;
            }
            int n = 0, p = 0;
            if (scaling && oracle_scale_factor(mx, target, &n, &p) != 0) { status = -1; n = 0; p = 0; }
            codes_out[(size_t)co * 16 + pos] = (uint8_t)oracle_encode_code(n, p);
            for (int ci = 0; ci < Cin; ci++) {
                int64_t v = Wt[(size_t)ci * 16 + pos];
                size_t o = ((size_t)co * Cin + ci) * 16 + pos;
                if (W_out) W_out[o] = v;
                Wp_out[o] = n ? oracle_rha_shift(v * n, p) : v;
            }
        }
    }
    free(Wt);
    return status;
}

/* F(2x2) input transform of every tile: D_out [T][Cin][16], T = N*th*tw with
 * th = ceil(Ho/2), patch origin (2ty - pad, 2tx - pad).                    */
void oracle_input_transform2_16(const int16_t *x, int N, int H, int W, int Cin, int pad, int layout,
                                int64_t *D_out) {
    int Ho = H + 2 * pad - 2, Wo = W + 2 * pad - 2;
    int th = (Ho + 1) / 2, tw = (Wo + 1) / 2;
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; n++)
        for (int ty = 0; ty < th; ty++)
            for (int tx = 0; tx < tw; tx++)
                for (int ci = 0; ci < Cin; ci++) {
                    int64_t d[4][4], D[4][4];
                    for (int a = 0; a < 4; a++)
                        for (int b = 0; b < 4; b++)
                            d[a][b] = x_at(x, layout, N, Cin, H, W, n, ci, 2 * ty - pad + a, 2 * tx - pad + b);
                    oracle_input_tile2(d, D);
                    size_t t = ((size_t)n * th + ty) * tw + tx;
                    for (int pos = 0; pos < 16; pos++) D_out[(t * Cin + ci) * 16 + pos] = D[pos / 4][pos % 4];
                }
}

/* The F(2x2) pipeline end to end: as oracle_wino_conv with 2x2 output tiles,
 * out32 = rha(Y / 4).  M_out / Mpp_out [T][Cout][16] (may be NULL).
 * Returns 0; -1 scale-factor range; -3 unscaled and 4 does not divide Y;
 * -4 int32 range.                                                          */
int oracle_wino2_conv16(const int16_t *x, const int16_t *w, int N, int H, int W, int Cin, int Cout,
                        int pad, int layout, int scaling, int target, int32_t M0, int S,
                        int32_t *out32, int8_t *y8, int64_t *M_out, int64_t *Mpp_out) {
    int Ho = H + 2 * pad - 2, Wo = W + 2 * pad - 2;
    int th = (Ho + 1) / 2, tw = (Wo + 1) / 2;
    size_t T = (size_t)N * th * tw;
    int status = 0;
    int64_t *Wp = (int64_t *)malloc(sizeof(int64_t) * 16 * (size_t)Cout * (Cin > 0 ? Cin : 1));
    uint8_t *codes = (uint8_t *)malloc((size_t)Cout * 16);
    int64_t *D = (int64_t *)malloc(sizeof(int64_t) * 16 * T * (Cin > 0 ? Cin : 1));
    if (oracle_filter_transform2_16(w, Cout, Cin, layout, scaling, target, NULL, Wp, codes) != 0) status = -1;
    oracle_input_transform2_16(x, N, H, W, Cin, pad, layout, D);
    int bad_div = 0, bad_range = 0;
#pragma omp parallel for collapse(2) schedule(dynamic) reduction(| : bad_div, bad_range)
    for (long long t = 0; t < (long long)T; t++)
        for (int co = 0; co < Cout; co++) {
            int64_t M[4][4], Mpp[4][4];
            memset(M, 0, sizeof(M));
            for (int ci = 0; ci < Cin; ci++)             /* Hadamard products over channels */
                for (int pos = 0; pos < 16; pos++)
                    M[pos / 4][pos % 4] += Wp[((size_t)co * Cin + ci) * 16 + pos] * D[((size_t)t * Cin + ci) * 16 + pos];
            for (int pos = 0; pos < 16; pos++) {          /* reverse scaling */
                int64_t v = M[pos / 4][pos % 4];
                int n, p, m = 0, q = 0;
                oracle_decode_code(codes[(size_t)co * 16 + pos], &n, &p);
                if (n) { oracle_reverse_factor(n, p, &m, &q); v = oracle_rha_shift(v * m, q); }
                Mpp[pos / 4][pos % 4] = v;
                if (v > INT32_MAX || v < INT32_MIN) bad_range = 1;
                if (M_out) M_out[((size_t)t * Cout + co) * 16 + pos] = M[pos / 4][pos % 4];
                if (Mpp_out) Mpp_out[((size_t)t * Cout + co) * 16 + pos] = v;
            }
            int64_t Y[2][2];
            oracle_output_tile2(Mpp, Y);
            int n_img = (int)(t / ((size_t)th * tw));
            int rem = (int)(t % ((size_t)th * tw));
            int ty = rem / tw, tx = rem % tw;
            for (int i = 0; i < 2; i++)
                for (int j = 0; j < 2; j++) {
                    if (Y[i][j] > INT32_MAX || Y[i][j] < INT32_MIN) bad_range = 1;
                    if (!scaling && (Y[i][j] % 4) != 0) bad_div = 1;
                    int oy = 2 * ty + i, ox = 2 * tx + j;
                    if (oy >= Ho || ox >= Wo) continue;
                    int64_t o32 = oracle_rha_shift(Y[i][j], OUT2_DIV_SHIFT);
                    int64_t yi = y_index(layout, Cout, Ho, Wo, n_img, co, oy, ox);
                    out32[yi] = (int32_t)o32;
                    if (y8) {
                        int64_t r = oracle_rha_shift(o32 * (int64_t)M0, S);
                        if (r > 127) r = 127;
                        if (r < -128) r = -128;
                        y8[yi] = (int8_t)r;
                    }
                }
        }
    if (bad_range) status = status ? status : -4;
    if (bad_div) status = status ? status : -3;
    free(Wp); free(codes); free(D);
    return status;
}

/* Requantisation alone (O12), for direct-conv references. */
void oracle_requant(const int64_t *v, int64_t count, int32_t M0, int S, int8_t *y8) {
    for (int64_t i = 0; i < count; i++) {
        int64_t r = oracle_rha_shift(v[i] * (int64_t)M0, S);
        if (r > 127) r = 127;
        if (r < -128) r = -128;
        y8[i] = (int8_t)r;
    }
}

/* 2x2 stride-2 max pool on int8 (harness for the VGG stack, A22). */
void oracle_maxpool2(const int8_t *x, int N, int H, int W, int C, int layout, int8_t *y) {
    int Ho = H / 2, Wo = W / 2;
    for (int n = 0; n < N; n++)
        for (int c = 0; c < C; c++)
            for (int oy = 0; oy < Ho; oy++)
                for (int ox = 0; ox < Wo; ox++) {
                    int m = -128;
                    for (int a = 0; a < 2; a++)
                        for (int b = 0; b < 2; b++) {
                            int h = 2 * oy + a, w = 2 * ox + b;
                            int v = layout == 0 ? x[(((int64_t)n * C + c) * H + h) * W + w]
                                                : x[(((int64_t)n * H + h) * W + w) * C + c];
                            if (v > m) m = v;
                        }
                    if (layout == 0) y[(((int64_t)n * C + c) * Ho + oy) * Wo + ox] = (int8_t)m;
                    else y[(((int64_t)n * Ho + oy) * Wo + ox) * C + c] = (int8_t)m;
                }
}

/* Matrix accessors so tests can inspect what the oracle uses. */
void oracle_matrices(int *bt_re, int *bt_im, int *g4_re, int *g4_im, int *at_re, int *at_im) {
    memcpy(bt_re, BT_RE, sizeof(BT_RE)); memcpy(bt_im, BT_IM, sizeof(BT_IM));
    memcpy(g4_re, G4_RE, sizeof(G4_RE)); memcpy(g4_im, G4_IM, sizeof(G4_IM));
    memcpy(at_re, AT_RE, sizeof(AT_RE)); memcpy(at_im, AT_IM, sizeof(AT_IM));
}

/* Thin wrappers over single tiles (int64 arrays) for ctypes callers. */
void oracle_filter_tile64(const int64_t *g9, int64_t *W72) {
    int64_t g[3][3]; gint W[6][6];
    for (int i = 0; i < 9; i++) g[i / 3][i % 3] = g9[i];
    oracle_filter_tile(g, W);
    for (int p = 0; p < 36; p++) { W72[2 * p] = W[p / 6][p % 6].re; W72[2 * p + 1] = W[p / 6][p % 6].im; }
}
void oracle_input_tile64(const int64_t *d36, int64_t *D72) {
    int64_t d[6][6]; gint D[6][6];
    for (int i = 0; i < 36; i++) d[i / 6][i % 6] = d36[i];
    oracle_input_tile(d, D);
    for (int p = 0; p < 36; p++) { D72[2 * p] = D[p / 6][p % 6].re; D72[2 * p + 1] = D[p / 6][p % 6].im; }
}
int oracle_output_tile64(const int64_t *M72, int64_t *Y16) {
    gint M[6][6]; int64_t Y[4][4];
    for (int p = 0; p < 36; p++) { M[p / 6][p % 6].re = M72[2 * p]; M[p / 6][p % 6].im = M72[2 * p + 1]; }
    int r = oracle_output_tile((const gint(*)[6])M, Y);
    for (int i = 0; i < 16; i++) Y16[i] = Y[i / 4][i % 4];
    return r;
}

/* ---- entry points on int8 tensors (widened to int16) and on uint8 tensors with
 * zero points (f2: the paper's affine uint8 model: values x - zx, w - zw
 * in [-255, 255]; padding is the real value 0, i.e. x - zx = 0).           */
static int16_t *widen8(const int8_t *a, size_t n) {
    int16_t *r = (int16_t *)malloc(sizeof(int16_t) * (n ? n : 1));
    for (size_t i = 0; i < n; i++) r[i] = a[i];
    return r;
}
static int16_t *widen_u8(const uint8_t *a, size_t n, int z) {
    int16_t *r = (int16_t *)malloc(sizeof(int16_t) * (n ? n : 1));
    for (size_t i = 0; i < n; i++) r[i] = (int16_t)((int)a[i] - z);
    return r;
}
#define XN ((size_t)N * H * W * Cin)
#define WN ((size_t)Cout * Cin * 9)

void oracle_direct_conv(const int8_t *x, const int8_t *w, int N, int H, int W,
                        int Cin, int Cout, int pad, int layout, int64_t *out) {
    int16_t *x16 = widen8(x, XN), *w16 = widen8(w, WN);
    oracle_direct_conv16(x16, w16, N, H, W, Cin, Cout, pad, layout, out);
    free(x16); free(w16);
}
int oracle_filter_transform(const int8_t *w, int Cout, int Cin, int layout, int scaling,
                            int target, int64_t *W_out, int64_t *Wp_out, uint8_t *codes_out) {
    int16_t *w16 = widen8(w, WN);
    int r = oracle_filter_transform16(w16, Cout, Cin, layout, scaling, target, W_out, Wp_out, codes_out);
    free(w16);
    return r;
}
void oracle_input_transform(const int8_t *x, int N, int H, int W, int Cin, int pad,
                            int layout, int64_t *D_out) {
    int16_t *x16 = widen8(x, XN);
    oracle_input_transform16(x16, N, H, W, Cin, pad, layout, D_out);
    free(x16);
}
int oracle_wino_conv(const int8_t *x, const int8_t *w, int N, int H, int W, int Cin, int Cout,
                     int pad, int layout, int scaling, int target, int32_t M0, int S,
                     int32_t *out32, int8_t *y8, int64_t *M_out, int64_t *Mpp_out) {
    int16_t *x16 = widen8(x, XN), *w16 = widen8(w, WN);
    int r = oracle_wino_conv16(x16, w16, N, H, W, Cin, Cout, pad, layout, scaling, target, M0, S,
                               out32, y8, M_out, Mpp_out);
    free(x16); free(w16);
    return r;
}
int oracle_filter_transform2(const int8_t *w, int Cout, int Cin, int layout, int scaling, int target,
                             int64_t *W_out, int64_t *Wp_out, uint8_t *codes_out) {
    int16_t *w16 = widen8(w, WN);
    int r = oracle_filter_transform2_16(w16, Cout, Cin, layout, scaling, target, W_out, Wp_out, codes_out);
    free(w16);
    return r;
}
void oracle_input_transform2(const int8_t *x, int N, int H, int W, int Cin, int pad, int layout,
                             int64_t *D_out) {
    int16_t *x16 = widen8(x, XN);
    oracle_input_transform2_16(x16, N, H, W, Cin, pad, layout, D_out);
    free(x16);
}
int oracle_wino2_conv(const int8_t *x, const int8_t *w, int N, int H, int W, int Cin, int Cout,
                      int pad, int layout, int scaling, int target, int32_t M0, int S,
                      int32_t *out32, int8_t *y8, int64_t *M_out, int64_t *Mpp_out) {
    int16_t *x16 = widen8(x, XN), *w16 = widen8(w, WN);
    int r = oracle_wino2_conv16(x16, w16, N, H, W, Cin, Cout, pad, layout, scaling, target, M0, S,
                                out32, y8, M_out, Mpp_out);
    free(x16); free(w16);
    return r;
}
/* uint8 + zero points (f2) */
void oracle_direct_conv_u8(const uint8_t *x, const uint8_t *w, int zx, int zw, int N, int H, int W,
                           int Cin, int Cout, int pad, int layout, int64_t *out) {
    int16_t *x16 = widen_u8(x, XN, zx), *w16 = widen_u8(w, WN, zw);
    oracle_direct_conv16(x16, w16, N, H, W, Cin, Cout, pad, layout, out);
    free(x16); free(w16);
}
int oracle_filter_transform_u8(const uint8_t *w, int zw, int Cout, int Cin, int layout, int scaling, int target,
                               int64_t *W_out, int64_t *Wp_out, uint8_t *codes_out) {
    int16_t *w16 = widen_u8(w, WN, zw);
    int r = oracle_filter_transform16(w16, Cout, Cin, layout, scaling, target, W_out, Wp_out, codes_out);
    free(w16);
    return r;
}
void oracle_input_transform_u8(const uint8_t *x, int zx, int N, int H, int W, int Cin, int pad, int layout,
                               int64_t *D_out) {
    int16_t *x16 = widen_u8(x, XN, zx);
    oracle_input_transform16(x16, N, H, W, Cin, pad, layout, D_out);
    free(x16);
}
int oracle_wino_conv_u8(const uint8_t *x, const uint8_t *w, int zx, int zw, int N, int H, int W, int Cin,
                        int Cout, int pad, int layout, int scaling, int target, int32_t M0, int S,
                        int32_t *out32, int8_t *y8, int64_t *M_out, int64_t *Mpp_out) {
    int16_t *x16 = widen_u8(x, XN, zx), *w16 = widen_u8(w, WN, zw);
    int r = oracle_wino_conv16(x16, w16, N, H, W, Cin, Cout, pad, layout, scaling, target, M0, S,
                               out32, y8, M_out, Mpp_out);
    free(x16); free(w16);
    return r;
}
/* the rational F(2x2) pipeline on uint8 tensors with zero points (f1 x f2: the paper's own evaluated
 * configuration) -- the same int16 core as the int8 entry points                    */
int oracle_filter_transform2_u8(const uint8_t *w, int zw, int Cout, int Cin, int layout, int scaling, int target,
                                int64_t *W_out, int64_t *Wp_out, uint8_t *codes_out) {
    int16_t *w16 = widen_u8(w, WN, zw);
    int r = oracle_filter_transform2_16(w16, Cout, Cin, layout, scaling, target, W_out, Wp_out, codes_out);
    free(w16);
    return r;
}
void oracle_input_transform2_u8(const uint8_t *x, int zx, int N, int H, int W, int Cin, int pad, int layout,
                                int64_t *D_out) {
    int16_t *x16 = widen_u8(x, XN, zx);
    oracle_input_transform2_16(x16, N, H, W, Cin, pad, layout, D_out);
    free(x16);
}
int oracle_wino2_conv_u8(const uint8_t *x, const uint8_t *w, int zx, int zw, int N, int H, int W, int Cin,
                         int Cout, int pad, int layout, int scaling, int target, int32_t M0, int S,
                         int32_t *out32, int8_t *y8, int64_t *M_out, int64_t *Mpp_out) {
    int16_t *x16 = widen_u8(x, XN, zx), *w16 = widen_u8(w, WN, zw);
    int r = oracle_wino2_conv16(x16, w16, N, H, W, Cin, Cout, pad, layout, scaling, target, M0, S,
                                out32, y8, M_out, Mpp_out);
    free(x16); free(w16);
    return r;
}
#undef XN
#undef WN

