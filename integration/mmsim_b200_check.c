/* integration/mmsim_b200_check.c — a plain C client of the reference's public header
 * (proj/include/mmsim.h) linked against libmmsim_b200.so: the reference library with the
 * b200 backend. Selecting `backend = b200` in a config must give the reference's results
 * through every verb a C user has:
 *   1. config parse / describe round trip keeps `backend = b200`        (capi.cpp:106-143)
 *   2. mmsim_sim_create/step/average/energy/max_torque/run, b200 vs serial (capi.cpp:145-239)
 *   3. mmsim_simulate writes the same trajectory TSV as the serial backend (capi.cpp:241-260)
 *   4. mmsim_benchmark renders b200 columns next to serial             (capi.cpp:262-284)
 *   5. unknown backends are still rejected
 * Usage: mmsim_b200_check <scratch dir>. Exit 0 = pass, 1 = mismatch, 2 = no usable GPU. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mmsim.h"

static int failures = 0;

#define EXPECT(cond, ...)                                  \
    do {                                                   \
        if (!(cond)) {                                     \
            printf("FAIL %s:%d: ", __FILE__, __LINE__);    \
            printf(__VA_ARGS__);                           \
            printf("\n");                                  \
            ++failures;                                    \
        }                                                  \
    } while (0)

static mmsim_config* parse(const char* text) {
    mmsim_config* cfg = NULL;
    int rc = mmsim_config_parse(text, &cfg);
    if (rc != MMSIM_OK) {
        printf("config parse failed (%s): %s\n", mmsim_status_string(rc), mmsim_last_error());
        exit(1);
    }
    return cfg;
}

typedef struct {
    long long step[64];
    double m[64][3];
    int n;
} records;

static void sink(void* user, long long step, double mx, double my, double mz) {
    records* r = (records*)user;
    if (r->n < 64) {
        r->step[r->n] = step;
        r->m[r->n][0] = mx;
        r->m[r->n][1] = my;
        r->m[r->n][2] = mz;
        ++r->n;
    }
}

static int read_tsv(const char* path, long long* steps, double (*m)[3], int cap) {
    FILE* f = fopen(path, "rb");
    if (!f) return -1;
    int n = 0;
    while (n < cap && fscanf(f, "%lld %lf %lf %lf", &steps[n], &m[n][0], &m[n][1], &m[n][2]) == 4) ++n;
    fclose(f);
    return n;
}

int main(int argc, char** argv) {
    const char* dir = argc > 1 ? argv[1] : ".";
    char text[1024], path_b200[512], path_serial[512];
    snprintf(path_b200, sizeof path_b200, "%s/traj_b200.tsv", dir);
    snprintf(path_serial, sizeof path_serial, "%s/traj_serial.tsv", dir);

    /* ---- 1. config round trip */
    const char* body = "problem = sp4\nprecision = f64\nsteps = 600\ncadence = 100\n";
    snprintf(text, sizeof text, "%sbackend = b200\n", body);
    mmsim_config* cfg_b = parse(text);
    snprintf(text, sizeof text, "%sbackend = serial\n", body);
    mmsim_config* cfg_s = parse(text);
    char* desc = NULL;
    EXPECT(mmsim_config_describe(cfg_b, &desc) == MMSIM_OK, "describe: %s", mmsim_last_error());
    EXPECT(desc && strstr(desc, "backend = b200\n"), "describe lost the backend:\n%s", desc ? desc : "");
    mmsim_config* again = desc ? parse(desc) : NULL;
    mmsim_string_free(desc);

    /* ---- 2. handle API on both backends */
    mmsim_sim *sb = NULL, *ss = NULL;
    int rc = mmsim_sim_create(again ? again : cfg_b, &sb);
    if (rc != MMSIM_OK) {
        printf("b200 sim_create failed (%s): %s\n", mmsim_status_string(rc), mmsim_last_error());
        return strstr(mmsim_last_error(), "CUDA") || strstr(mmsim_last_error(), "cuda") ? 2 : 1;
    }
    EXPECT(mmsim_sim_create(cfg_s, &ss) == MMSIM_OK, "serial sim_create: %s", mmsim_last_error());
    EXPECT(mmsim_sim_step(sb, 25) == MMSIM_OK && mmsim_sim_step(ss, 25) == MMSIM_OK, "step: %s",
           mmsim_last_error());
    long long ib = -1, is = -2;
    mmsim_sim_step_index(sb, &ib);
    mmsim_sim_step_index(ss, &is);
    EXPECT(ib == 25 && is == 25, "step_index %lld vs %lld", ib, is);
    double ab[3], as[3], eb, es, tb, ts;
    mmsim_sim_average(sb, ab);
    mmsim_sim_average(ss, as);
    for (int c = 0; c < 3; ++c) EXPECT(fabs(ab[c] - as[c]) <= 1e-12, "average[%d] %.17g vs %.17g", c, ab[c], as[c]);
    EXPECT(mmsim_sim_energy(sb, &eb) == MMSIM_OK && mmsim_sim_energy(ss, &es) == MMSIM_OK, "energy");
    EXPECT(fabs(eb - es) <= 1e-9 * fabs(es), "energy %.17g vs %.17g", eb, es);
    EXPECT(mmsim_sim_max_torque(sb, &tb) == MMSIM_OK && mmsim_sim_max_torque(ss, &ts) == MMSIM_OK, "torque");
    EXPECT(fabs(tb - ts) <= 1e-9 * fabs(ts), "max_torque %.17g vs %.17g", tb, ts);
    records rb = {{0}, {{0}}, 0}, rs = {{0}, {{0}}, 0};
    long long db = 0, ds = 0;
    EXPECT(mmsim_sim_run(sb, 40, 10, sink, &rb, &db) == MMSIM_OK, "run b200: %s", mmsim_last_error());
    EXPECT(mmsim_sim_run(ss, 40, 10, sink, &rs, &ds) == MMSIM_OK, "run serial: %s", mmsim_last_error());
    EXPECT(db == 40 && ds == 40 && rb.n == rs.n && rb.n == 4, "run records %d/%d done %lld/%lld", rb.n, rs.n, db, ds);
    for (int i = 0; i < rb.n && i < rs.n; ++i) {
        EXPECT(rb.step[i] == rs.step[i], "record step %lld vs %lld", rb.step[i], rs.step[i]);
        for (int c = 0; c < 3; ++c)
            EXPECT(fabs(rb.m[i][c] - rs.m[i][c]) <= 1e-12, "record %d comp %d: %.17g vs %.17g", i, c, rb.m[i][c],
                   rs.m[i][c]);
    }
    mmsim_sim_free(sb);
    mmsim_sim_free(ss);

    /* ---- 3. whole-run verb: identical trajectory files */
    EXPECT(mmsim_simulate(cfg_b, path_b200) == MMSIM_OK, "simulate b200: %s", mmsim_last_error());
    EXPECT(mmsim_simulate(cfg_s, path_serial) == MMSIM_OK, "simulate serial: %s", mmsim_last_error());
    long long stb[16], sts[16];
    double mb[16][3], msr[16][3];
    const int nb = read_tsv(path_b200, stb, mb, 16), ns = read_tsv(path_serial, sts, msr, 16);
    EXPECT(nb == 6 && ns == 6, "trajectory rows %d / %d", nb, ns);
    for (int i = 0; i < nb && i < ns; ++i) {
        EXPECT(stb[i] == sts[i], "trajectory step %lld vs %lld", stb[i], sts[i]);
        /* 6 printed decimals: values 1e-13 apart may round one ulp of the format apart */
        for (int c = 0; c < 3; ++c)
            EXPECT(fabs(mb[i][c] - msr[i][c]) <= 1.5e-6, "trajectory row %d comp %d", i, c);
    }

    /* ---- 4. benchmark table with b200 columns */
    char *table = NULL, *tsv = NULL;
    EXPECT(mmsim_benchmark("8,16", "serial,b200", "f64", 1, 3, &table, &tsv) == MMSIM_OK, "benchmark: %s",
           mmsim_last_error());
    EXPECT(table && strstr(table, "b200 f64 (ms)") && strstr(table, "Speedup"), "table:\n%s", table ? table : "");
    EXPECT(tsv && strstr(tsv, "16^3\tb200\tf64\t") && !strstr(tsv, "nan"), "tsv:\n%s", tsv ? tsv : "");
    if (table) printf("%s", table);
    mmsim_string_free(table);
    mmsim_string_free(tsv);

    /* ---- 5. still strict about names */
    mmsim_config* badcfg = NULL;
    EXPECT(mmsim_config_parse("problem = sp4\nbackend = gpu\n", &badcfg) != MMSIM_OK, "backend = gpu accepted");
    EXPECT(strstr(mmsim_last_error(), "b200") != NULL, "error does not list b200: %s", mmsim_last_error());

    mmsim_config_free(cfg_b);
    mmsim_config_free(cfg_s);
    mmsim_config_free(again);
    printf(failures ? "mmsim b200 check: %d failure(s)\n" : "mmsim b200 check: ok\n", failures);
    return failures ? 1 : 0;
}
