timeout 120 python tools/tile_roles.py 4096 4096
