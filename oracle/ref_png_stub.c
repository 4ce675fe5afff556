/* Test infrastructure: refusing definitions for the libpng shim
 * (oracle/shim_png/png.h).  Only the scene-file half of io.cpp is exercised. */
#include "png.h"
#include <stdlib.h>
int png_sig_cmp(png_const_bytep s, size_t a, size_t b) { (void)s; (void)a; (void)b; return 1; }
png_structp png_create_read_struct(png_const_charp v, png_voidp e, png_error_ptr f, png_error_ptr w) {
  (void)v; (void)e; (void)f; (void)w; return NULL; }
png_structp png_create_write_struct(png_const_charp v, png_voidp e, png_error_ptr f, png_error_ptr w) {
  (void)v; (void)e; (void)f; (void)w; return NULL; }
png_infop png_create_info_struct(png_structp p) { (void)p; return NULL; }
void png_destroy_read_struct(png_structpp p, png_infopp i, png_infopp e) { (void)p; (void)i; (void)e; }
void png_destroy_write_struct(png_structpp p, png_infopp i) { (void)p; (void)i; }
jmp_buf* png_shim_jmpbuf(png_structp p) { (void)p; abort(); }
void png_init_io(png_structp p, FILE* fp) { (void)p; (void)fp; abort(); }
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
  (void)p; (void)i; (void)w; (void)h; (void)bd; (void)ct; (void)il; (void)cm; (void)fm; abort(); }
void png_write_info(png_structp p, png_infop i) { (void)p; (void)i; abort(); }
void png_write_row(png_structp p, png_const_bytep r) { (void)p; (void)r; abort(); }
void png_write_end(png_structp p, png_infop i) { (void)p; (void)i; abort(); }
