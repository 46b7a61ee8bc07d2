/*
 * oracle/ccl_oracle.c -- CPU oracle for 2D binary-image connected-components
 * labeling.  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_1708_08180_b200/csrc) and neither side includes the other.
 *
 * What is computed (the plain definition; SURVEY.md §8(c) "Definition"):
 *   idx(x,y) = y*W + x                       (raster order)
 *   fg(p)   <=> img[p] != 0                  (reading P1 of DESIGN.md)
 *   N4(x,y) = {(x+-1,y),(x,y+-1)} clipped, no wrap   (PAPER.md:209, 4-conn)
 *   N8      = N4 u {(x+-1,y+-1)} clipped               (north_star 8-conn)
 *   L[p] = 0 if !fg(p), else 1 + min{ idx(q) : q in p's component }
 * "CCL ... give[s] a unique ID to each connected region"; the
 * unique ID chosen is the component's minimum raster index + 1 (north_star
 * canonical form; min-label convergence of SPEC.md:135, :140).
 *
 * Two independent algorithms, sharing nothing with each other either:
 *   O1 oracle_bfs      -- raster-order seeded flood fill with an explicit stack
 *                         (SPEC.md:363-366).  The first unlabeled foreground
 *                         pixel met in raster order is its component's minimum,
 *                         so the output is canonical by construction.
 *   O2 oracle_twopass  -- sequential two-pass union-find: pass 1 unions each
 *                         foreground pixel with its already-visited foreground
 *                         neighbours (W,N for 4-conn; W,NW,N,NE for 8-conn) by
 *                         minimum root (SPEC.md:115-123 union_min, SPEC.md:140
 *                         "union by minimum root"); pass 2 writes find(p)+1
 *                         (SPEC.md:124-127 flatten).
 *
 * Return codes: 0 ok, 1 null pointer, 2 bad dims, 3 too large (H*W > 2^31-1),
 * 4 bad connectivity, 5 out of host memory.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define O_OK 0
#define O_ERR_NULL 1
#define O_ERR_DIMS 2
#define O_ERR_TOO_LARGE 3
#define O_ERR_CONN 4
#define O_ERR_NOMEM 5

static int check_args(const uint8_t* img, int64_t H, int64_t W, int conn, const int32_t* out) {
    if (!img || !out) return O_ERR_NULL;
    if (H < 1 || W < 1) return O_ERR_DIMS;
    if (H > INT32_MAX / W) return O_ERR_TOO_LARGE;
    if (conn != 4 && conn != 8) return O_ERR_CONN;
    return O_OK;
}

/* O1: flood fill. */
int oracle_bfs(const uint8_t* img, int64_t H, int64_t W, int conn, int32_t* out) {
    int rc = check_args(img, H, W, conn, out);
    if (rc) return rc;
    const int64_t n = H * W;
    memset(out, 0, (size_t)n * sizeof(int32_t));
    int32_t* stack = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    if (!stack) return O_ERR_NOMEM;
    for (int64_t s = 0; s < n; ++s) {
        if (img[s] == 0 || out[s] != 0) continue;
        const int32_t lab = (int32_t)(s + 1);
        int64_t top = 0;
        out[s] = lab;
        stack[top++] = (int32_t)s;
        while (top > 0) {
            const int64_t p = stack[--top];
            const int64_t y = p / W, x = p % W;
            for (int64_t dy = -1; dy <= 1; ++dy) {
                for (int64_t dx = -1; dx <= 1; ++dx) {
                    if (dy == 0 && dx == 0) continue;
                    if (conn == 4 && dy != 0 && dx != 0) continue;
                    const int64_t yy = y + dy, xx = x + dx;
                    if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
                    const int64_t q = yy * W + xx;
                    if (img[q] != 0 && out[q] == 0) {
                        out[q] = lab;
                        stack[top++] = (int32_t)q;
                    }
                }
            }
        }
    }
    free(stack);
    return O_OK;
}

/* Equal-value mode (the paper's raw-value tests
 * dBuff[tid] == dBuff[tid-1], and the
 * SPEC CPU program's semantics): every pixel, background
 * included, belongs to the component of equal-valued neighbours; its label is
 * the component's minimum raster index, 0-based.  Flood
 * fill in raster order as O1, with "same value" instead of "both nonzero". */
int oracle_bfs_equal(const uint8_t* img, int64_t H, int64_t W, int conn, int32_t* out) {
    int rc = check_args(img, H, W, conn, out);
    if (rc) return rc;
    const int64_t n = H * W;
    for (int64_t i = 0; i < n; ++i) out[i] = -1;
    int32_t* stack = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    if (!stack) return O_ERR_NOMEM;
    for (int64_t s = 0; s < n; ++s) {
        if (out[s] >= 0) continue;
        const uint8_t v = img[s];
        int64_t top = 0;
        out[s] = (int32_t)s;
        stack[top++] = (int32_t)s;
        while (top > 0) {
            const int64_t p = stack[--top];
            const int64_t y = p / W, x = p % W;
            for (int64_t dy = -1; dy <= 1; ++dy) {
                for (int64_t dx = -1; dx <= 1; ++dx) {
                    if (dy == 0 && dx == 0) continue;
                    if (conn == 4 && dy != 0 && dx != 0) continue;
                    const int64_t yy = y + dy, xx = x + dx;
                    if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
                    const int64_t q = yy * W + xx;
                    if (img[q] == v && out[q] < 0) {
                        out[q] = (int32_t)s;
                        stack[top++] = (int32_t)q;
                    }
                }
            }
        }
    }
    free(stack);
    return O_OK;
}

/* 3D volumes ("2D/3D grid"): voxel
 * (x,y,z) of a D x H x W volume has raster index (z*H + y)*W + x; foreground
 * = nonzero; 6-connectivity (faces) or 26-connectivity (faces, edges,
 * corners), clipped; label = 0 or 1 + the component's minimum raster index.
 * Flood fill seeded in raster order, as O1. */
int oracle_bfs3d(const uint8_t* vol, int64_t D, int64_t H, int64_t W, int conn, int32_t* out) {
    if (!vol || !out) return O_ERR_NULL;
    if (D < 1 || H < 1 || W < 1) return O_ERR_DIMS;
    if (H * W > INT32_MAX / D) return O_ERR_TOO_LARGE;
    if (conn != 6 && conn != 26) return O_ERR_CONN;
    const int64_t n = D * H * W;
    memset(out, 0, (size_t)n * sizeof(int32_t));
    int32_t* stack = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    if (!stack) return O_ERR_NOMEM;
    for (int64_t s = 0; s < n; ++s) {
        if (vol[s] == 0 || out[s] != 0) continue;
        const int32_t lab = (int32_t)(s + 1);
        int64_t top = 0;
        out[s] = lab;
        stack[top++] = (int32_t)s;
        while (top > 0) {
            const int64_t p = stack[--top];
            const int64_t z = p / (H * W), y = (p / W) % H, x = p % W;
            for (int64_t dz = -1; dz <= 1; ++dz)
                for (int64_t dy = -1; dy <= 1; ++dy)
                    for (int64_t dx = -1; dx <= 1; ++dx) {
                        const int64_t nz = (dz != 0) + (dy != 0) + (dx != 0);
                        if (nz == 0 || (conn == 6 && nz != 1)) continue;
                        const int64_t zz = z + dz, yy = y + dy, xx = x + dx;
                        if (zz < 0 || zz >= D || yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
                        const int64_t q = (zz * H + yy) * W + xx;
                        if (vol[q] != 0 && out[q] == 0) {
                            out[q] = lab;
                            stack[top++] = (int32_t)q;
                        }
                    }
        }
    }
    free(stack);
    return O_OK;
}

/* O2: sequential two-pass union-find with minimum-root union. */
static int64_t tp_find(int32_t* parent, int64_t a) {
    while (parent[a] != a) {
        parent[a] = parent[parent[a]]; /* path halving: writes an ancestor */
        a = parent[a];
    }
    return a;
}

static void tp_union_min(int32_t* parent, int64_t a, int64_t b) {
    a = tp_find(parent, a);
    b = tp_find(parent, b);
    if (a == b) return;
    if (a < b) parent[b] = (int32_t)a; /* larger root under smaller */
    else parent[a] = (int32_t)b;
}

int oracle_twopass(const uint8_t* img, int64_t H, int64_t W, int conn, int32_t* out) {
    int rc = check_args(img, H, W, conn, out);
    if (rc) return rc;
    const int64_t n = H * W;
    int32_t* parent = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    if (!parent) return O_ERR_NOMEM;
    /* pass 1: raster scan, union with already-visited neighbours */
    for (int64_t y = 0; y < H; ++y) {
        for (int64_t x = 0; x < W; ++x) {
            const int64_t p = y * W + x;
            parent[p] = (int32_t)p;
            if (img[p] == 0) continue;
            if (x > 0 && img[p - 1]) tp_union_min(parent, p, p - 1);            /* W  */
            if (y > 0) {
                if (img[p - W]) tp_union_min(parent, p, p - W);                  /* N  */
                if (conn == 8) {
                    if (x > 0 && img[p - W - 1]) tp_union_min(parent, p, p - W - 1);     /* NW */
                    if (x + 1 < W && img[p - W + 1]) tp_union_min(parent, p, p - W + 1); /* NE */
                }
            }
        }
    }
    /* pass 2: every pixel <- root (+1), background 0 */
    for (int64_t p = 0; p < n; ++p)
        out[p] = img[p] ? (int32_t)(tp_find(parent, p) + 1) : 0;
    free(parent);
    return O_OK;
}

/* Batched: B independent images of H x W each (labels are per image). */
int oracle_bfs_batched(const uint8_t* img, int64_t B, int64_t H, int64_t W, int conn, int32_t* out) {
    if (B < 0) return O_ERR_DIMS;
    for (int64_t b = 0; b < B; ++b) {
        int rc = oracle_bfs(img + b * H * W, H, W, conn, out + b * H * W);
        if (rc) return rc;
    }
    return O_OK;
}
