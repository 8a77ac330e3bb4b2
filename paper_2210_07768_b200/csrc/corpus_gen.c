/* corpus_gen.c -- bulk synthetic corpus (measurement input), libfbxgen.so.
 *
 * Byte-identical restatement of corpus.make_corpus (itself byte-identical to
 * the reference generator corpus.py:52-143): one MT19937 stream seeded like
 * CPython's random.Random(int), drawn in the reference order -- driver rows,
 * then the profile side view, then basic payloads -- with CPython's
 * algorithms for random(), getrandbits/_randbelow, randint, choice, sample
 * (pool variant, n=16 <= setsize) and uniform.  JSON text is formatted like
 * json.dumps with the default separators.  Column images are written straight
 * into caller buffers in FBXC layout (null bitmaps LSB-first).
 */
#include <stdint.h>
#include <string.h>

/* ---- MT19937 (CPython _randommodule.c) --------------------------------- */
#define N 624
#define M 397
typedef struct { uint32_t mt[N]; int mti; } mt_t;

static void init_genrand(mt_t* s, uint32_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < N; i++)
    s->mt[i] = 1812433253u * (s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) + (uint32_t)i;
  s->mti = N;
}

static void init_by_array(mt_t* s, const uint32_t* key, int len) {
  init_genrand(s, 19650218u);
  int i = 1, j = 0;
  int k = N > len ? N : len;
  for (; k; k--) {
    s->mt[i] = (s->mt[i] ^ ((s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
    i++;
    j++;
    if (i >= N) { s->mt[0] = s->mt[N - 1]; i = 1; }
    if (j >= len) j = 0;
  }
  for (k = N - 1; k; k--) {
    s->mt[i] = (s->mt[i] ^ ((s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
    i++;
    if (i >= N) { s->mt[0] = s->mt[N - 1]; i = 1; }
  }
  s->mt[0] = 0x80000000u;
}

static uint32_t genrand(mt_t* s) {
  static const uint32_t mag01[2] = {0x0u, 0x9908b0dfu};
  uint32_t y;
  if (s->mti >= N) {
    int kk;
    for (kk = 0; kk < N - M; kk++) {
      y = (s->mt[kk] & 0x80000000u) | (s->mt[kk + 1] & 0x7fffffffu);
      s->mt[kk] = s->mt[kk + M] ^ (y >> 1) ^ mag01[y & 1u];
    }
    for (; kk < N - 1; kk++) {
      y = (s->mt[kk] & 0x80000000u) | (s->mt[kk + 1] & 0x7fffffffu);
      s->mt[kk] = s->mt[kk + (M - N)] ^ (y >> 1) ^ mag01[y & 1u];
    }
    y = (s->mt[N - 1] & 0x80000000u) | (s->mt[0] & 0x7fffffffu);
    s->mt[N - 1] = s->mt[M - 1] ^ (y >> 1) ^ mag01[y & 1u];
    s->mti = 0;
  }
  y = s->mt[s->mti++];
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= (y >> 18);
  return y;
}

static double rnd(mt_t* s) {
  uint32_t a = genrand(s) >> 5, b = genrand(s) >> 6;
  return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
}

static uint32_t getrandbits(mt_t* s, int k) { return k ? genrand(s) >> (32 - k) : 0u; }

static uint32_t below(mt_t* s, uint32_t n) { /* _randbelow_with_getrandbits */
  int k = 0;
  for (uint32_t t = n; t; t >>= 1) k++;
  uint32_t r = getrandbits(s, k);
  while (r >= n) r = getrandbits(s, k);
  return r;
}

static int64_t randint(mt_t* s, int64_t a, int64_t b) { return a + below(s, (uint32_t)(b - a + 1)); }

/* ---- corpus constants (corpus.py) --------------------------------------- */
static const char* VOCAB[16] = {"shoes", "running", "coffee", "beans", "noise", "cancelling",
                                "headphones", "mechanical", "keyboard", "standing", "desk",
                                "espresso", "grinder", "trail", "gravel", "bike"};
static const char* CITIES[11] = {"tokyo", "osaka", "kyoto", "sapporo", "nagoya", "fukuoka",
                                 "sendai", "hiroshima", "kobe", "yokohama", "unknown"};
static const char* BROKEN[4] = {"{\"u\": {\"city\": \"par", "{\"u\": [", "not json{", "{,}"};
static const char* SRC[2] = {"app", "web"};
static const uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;

static uint64_t fnv(const uint8_t* p, int n) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (int i = 0; i < n; i++) h = (h ^ p[i]) * 0x100000001B3ull;
  return h;
}

static void set_null(uint8_t* bm, uint64_t i) { bm[i >> 3] |= (uint8_t)(1u << (i & 7)); }

static int put(char* dst, const char* s) {
  int n = (int)strlen(s);
  memcpy(dst, s, (size_t)n);
  return n;
}

typedef struct {
  /* driver: instance_id, label, user_id, query, meta, age */
  int64_t *id, *label, *user, *age;
  uint8_t *id_n, *label_n, *user_n, *query_n, *meta_n, *age_n;
  uint32_t *query_off, *meta_off;
  uint8_t *query, *meta;
  /* profile: user_id, city, score (<= users rows) */
  int64_t* p_user;
  uint8_t *p_user_n, *p_city_n, *p_score_n;
  uint32_t* p_city_off;
  uint8_t* p_city;
  float* p_score;
  /* basic: instance_id, basic_a, basic_b, payload */
  int64_t *b_id, *b_a, *b_b;
  uint8_t *b_id_n, *b_a_n, *b_b_n, *b_pay_n;
  float* b_pay;
  uint64_t profile_rows; /* out */
} fbxgen_out;

/* Null bitmaps must be zeroed by the caller.  query/meta buffers: rows*48 and
 * rows*64 bytes are enough; p_city: users*16. */
int fbxgen_corpus(uint64_t rows, uint64_t users, uint64_t seed, int views, fbxgen_out* o) {
  mt_t st;
  uint32_t key[2];
  int klen = 0;
  key[0] = (uint32_t)seed;
  key[1] = (uint32_t)(seed >> 32);
  klen = key[1] ? 2 : 1;
  init_by_array(&st, key, klen);
  uint32_t qo = 0, mo = 0;
  o->query_off[0] = 0;
  o->meta_off[0] = 0;
  char tmp[256];
  for (uint64_t i = 0; i < rows; i++) {
    o->id[i] = (int64_t)(GOLDEN * (i + 1));
    o->label[i] = rnd(&st) < 0.3 ? 1 : 0;
    o->user[i] = (int64_t)below(&st, (uint32_t)users);
    if (rnd(&st) < 0.05) {
      set_null(o->query_n, i);
    } else {
      int k = (int)randint(&st, 1, 4);
      int pool[16];
      for (int q = 0; q < 16; q++) pool[q] = q;
      for (int q = 0; q < k; q++) {
        uint32_t j = below(&st, (uint32_t)(16 - q));
        if (q) o->query[qo++] = ' ';
        qo += (uint32_t)put((char*)o->query + qo, VOCAB[pool[j]]);
        pool[j] = pool[16 - q - 1];
      }
    }
    o->query_off[i + 1] = qo;
    double r = rnd(&st);
    if (r < 0.02) {
      mo += (uint32_t)put((char*)o->meta + mo, BROKEN[below(&st, 4)]);
    } else if (r < 0.05) {
      set_null(o->meta_n, i);
    } else if (r < 0.15) {
      int n = 0;
      n += put(tmp + n, "{\"src\": \"");
      n += put(tmp + n, SRC[below(&st, 2)]);
      n += put(tmp + n, "\"}");
      memcpy(o->meta + mo, tmp, (size_t)n);
      mo += (uint32_t)n;
    } else {
      const char* city = CITIES[below(&st, 11)];
      int tier = (int)randint(&st, 0, 3);
      const char* src = SRC[below(&st, 2)];
      int n = 0;
      n += put(tmp + n, "{\"u\": {\"city\": \"");
      n += put(tmp + n, city);
      n += put(tmp + n, "\", \"tier\": ");
      tmp[n++] = (char)('0' + tier);
      n += put(tmp + n, "}, \"src\": \"");
      n += put(tmp + n, src);
      n += put(tmp + n, "\"}");
      memcpy(o->meta + mo, tmp, (size_t)n);
      mo += (uint32_t)n;
    }
    o->meta_off[i + 1] = mo;
    r = rnd(&st);
    if (r < 0.10) {
      set_null(o->age_n, i);
      o->age[i] = 0;
    } else if (r < 0.15) {
      o->age[i] = randint(&st, 121, 190);
    } else {
      o->age[i] = randint(&st, 18, 90);
    }
  }
  uint64_t np = 0;
  if (views == 2) {
    uint32_t co = 0;
    o->p_city_off[0] = 0;
    for (uint64_t u = 0; u < users; u++) {
      if (rnd(&st) < 0.03) continue;
      o->p_user[np] = (int64_t)u;
      if (rnd(&st) < 0.04) {
        set_null(o->p_city_n, np);
      } else {
        co += (uint32_t)put((char*)o->p_city + co, CITIES[below(&st, 11)]);
      }
      o->p_city_off[np + 1] = co;
      if (rnd(&st) < 0.10) {
        set_null(o->p_score_n, np);
        o->p_score[np] = 0.0f;
      } else {
        o->p_score[np] = (float)(0.0 + (1.0 - 0.0) * rnd(&st));
      }
      np++;
    }
  }
  o->profile_rows = np;
  for (uint64_t i = 0; i < rows; i++) {
    uint64_t id = GOLDEN * (i + 1);
    uint8_t msg[9];
    memcpy(msg, &id, 8); /* little-endian host */
    o->b_id[i] = (int64_t)id;
    msg[8] = 'a';
    o->b_a[i] = (int64_t)fnv(msg, 9);
    msg[8] = 'b';
    o->b_b[i] = (int64_t)fnv(msg, 9);
    o->b_pay[i] = (float)(-1.0 + (1.0 - -1.0) * rnd(&st));
  }
  return 0;
}
