(kernel
  (param replications int)
  (param steps int)
  (param chunks int)
  (param posX array)
  (param posY array)
  (param out array)
  (local rid int)
  (local i int)
  (local u real)
  (local v real)
  (local d int)
  (local px real)
  (local py real)
  (body
    (assign rid (div (add tid.x (mul bdim.x (add tid.y (mul bdim.y (add tid.z (mul bdim.z (add bid.x (mul gdim.x bid.y)))))))) warpsize))
    (if (ne (mod (add tid.x (mul bdim.x (add tid.y (mul bdim.y tid.z)))) warpsize) 0)
      (then
        (halt)))
    (if (lt rid replications)
      (then
        (assign i 0)
        (while (lt i steps)
          (assign u (draw))
          (assign v (draw))
          (assign d (floor (mul 4.0 u)))
          (if (eq d 0)
            (then
              (load px posX rid)
              (store posX rid (add px 1.0)))
            (else
              (if (eq d 1)
                (then
                  (load px posX rid)
                  (store posX rid (sub px 1.0)))
                (else
                  (if (eq d 2)
                    (then
                      (load py posY rid)
                      (store posY rid (add py 1.0)))
                    (else
                      (load py posY rid)
                      (store posY rid (sub py 1.0))))))))
          (assign i (add i 1)))
        (load px posX rid)
        (store out rid (mod (add (mod px chunks) chunks) chunks))))))
