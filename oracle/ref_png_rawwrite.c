/* Test infrastructure: libpng shim (oracle/shim_png/png.h) whose write side
 * stores the rows uncompressed (a "RAWPNG w h" header + 8-bit RGB rows) so
 * that the reference acceptance suite's C10 criterion (acceptance.cpp:652-697,
 * which compares the bytes of two written images) is meaningful without
 * libpng: equal pixels <=> equal bytes.  The read side refuses, like
 * oracle/ref_png_stub.c.  Linked only into oracle/_ref/acceptance_*. */
#include "png.h"
#include <stdlib.h>
#include <string.h>

struct png_struct_def {
  jmp_buf jb;
  FILE* fp;
  png_uint_32 w, h;
};
struct png_info_def {
  int unused;
};

int png_sig_cmp(png_const_bytep s, size_t a, size_t b) { (void)s; (void)a; (void)b; return 1; }
png_structp png_create_read_struct(png_const_charp v, png_voidp e, png_error_ptr f, png_error_ptr w) {
  (void)v; (void)e; (void)f; (void)w; return NULL; }
png_structp png_create_write_struct(png_const_charp v, png_voidp e, png_error_ptr f, png_error_ptr w) {
  (void)v; (void)e; (void)f; (void)w;
  return (png_structp)calloc(1, sizeof(png_struct));
}
png_infop png_create_info_struct(png_structp p) { return p ? (png_infop)calloc(1, sizeof(png_info)) : NULL; }
void png_destroy_read_struct(png_structpp p, png_infopp i, png_infopp e) { (void)p; (void)i; (void)e; }
void png_destroy_write_struct(png_structpp p, png_infopp i) {
  if (i && *i) { free(*i); *i = NULL; }
  if (p && *p) { free(*p); *p = NULL; }
}
jmp_buf* png_shim_jmpbuf(png_structp p) { return &p->jb; }
void png_init_io(png_structp p, FILE* fp) { p->fp = fp; }
void png_set_sig_bytes(png_structp p, int n) { (void)p; (void)n; abort(); }
void png_read_info(png_structp p, png_infop i) { (void)p; (void)i; abort(); }
png_byte png_get_bit_depth(png_structp p, png_infop i) { (void)p; (void)i; abort(); }
png_byte png_get_color_type(png_structp p, png_infop i) { (void)p; (void)i; abort(); }
png_byte png_get_channels(png_structp p, png_infop i) { (void)p; (void)i; abort(); }
png_uint_32 png_get_image_width(png_structp p, png_infop i) { (void)p; (void)i; abort(); }
png_uint_32 png_get_image_height(png_structp p, png_infop i) { (void)p; (void)i; abort(); }
void png_set_expand(png_structp p) { (void)p; abort(); }
void png_set_packing(png_structp p) { (void)p; abort(); }
void png_set_gray_to_rgb(png_structp p) { (void)p; abort(); }
void png_read_update_info(png_structp p, png_infop i) { (void)p; (void)i; abort(); }
void png_read_row(png_structp p, png_bytep r, png_bytep d) { (void)p; (void)r; (void)d; abort(); }
void png_read_end(png_structp p, png_infop i) { (void)p; (void)i; abort(); }
void png_set_IHDR(png_structp p, png_infop i, png_uint_32 w, png_uint_32 h, int bd, int ct, int il, int cm, int fm) {
  (void)i; (void)bd; (void)ct; (void)il; (void)cm; (void)fm;
  p->w = w;
  p->h = h;
}
void png_write_info(png_structp p, png_infop i) {
  (void)i;
  fprintf(p->fp, "RAWPNG %u %u\n", p->w, p->h);
}
void png_write_row(png_structp p, png_const_bytep r) {
  if (fwrite(r, 1, (size_t)p->w * 3, p->fp) != (size_t)p->w * 3) longjmp(p->jb, 1);
}
void png_write_end(png_structp p, png_infop i) { (void)p; (void)i; }
